#!/bin/bash
# round-2 GPU check: TMEM probe, the GPU test suite, the bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 120 ./tools/tmem_probe > gpurun_out/r02a_tmem_probe.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/r02a_pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r02a_pytest_gpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
echo "bench exit $?" >> gpurun_out/r02a_bench.err
