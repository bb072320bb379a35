#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m "gpu and not slow" --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python tools/tune.py --configs ${1:-0,1,2,3,4} > gpurun_out/tune.jsonl 2> gpurun_out/tune.err; echo "tune rc=$?"; grep BEST gpurun_out/tune.jsonl
