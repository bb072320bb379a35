#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/r02d_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r02d_pytest.txt
timeout 600 python tools/small_scan.py > gpurun_out/r02d_small_scan.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
