#!/bin/bash
# round-2 re-entry: full GPU suite, bench (both arms) after the [half][plane][entry] layout
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02e_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r02e_pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r02e_pytest_gpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
echo "bench exit $?" >> gpurun_out/r02e_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02e_ref.json 2> gpurun_out/r02e_ref.err
echo "ref exit $?" >> gpurun_out/r02e_ref.err
