#!/bin/bash
# full check: GPU tests (not slow), planner vs tune on the headline configs, e2e chunk sweep, bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m "gpu and not slow" --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/tune.py --configs ${TUNE_CONFIGS:-1,2} > gpurun_out/tune.jsonl 2> gpurun_out/tune.err; echo "tune rc=$?"; grep BEST gpurun_out/tune.jsonl
timeout 600 python tools/e2e_chunks.py ${E2E_ARGS} > gpurun_out/e2e_chunks.txt 2>&1; echo "e2e rc=$?"; cat gpurun_out/e2e_chunks.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python tools/show_bench.py gpurun_out/bench.json 2>/dev/null | head -30
