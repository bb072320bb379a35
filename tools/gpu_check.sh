#!/bin/bash
# GPU pass: smoke, GPU tests (optionally incl. slow), short bench.  usage: bash tools/gpu_check.sh [slow]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out; rm -f gpurun_out/summary.txt
SEL="gpu and not slow"; [ "$1" == "slow" ] && SEL="gpu"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 2400 python -m pytest tests -q -m "$SEL" --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/summary.txt
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/summary.txt; tail -3 gpurun_out/bench.err
