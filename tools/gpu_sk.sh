#!/bin/bash
# stream-K check: parity tests for the forced stream-K path, then tune configs with stream-K included
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "streamk or every_compiled or medium" --timeout 600 -p no:cacheprovider > gpurun_out/pytest_sk.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_sk.log
timeout 1200 python tools/tune.py --configs ${1:-0,1,2,3} > gpurun_out/tune_sk.jsonl 2> gpurun_out/tune_sk.err; echo "tune rc=$?"; grep BEST gpurun_out/tune_sk.jsonl
