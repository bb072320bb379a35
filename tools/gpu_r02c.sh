#!/bin/bash
# bench with the new roofline / CPU baselines; e2e-first variant; sass mix committed
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
echo "bench exit $?" >> gpurun_out/r02c_bench.err
SG_BENCH_E2E_FIRST=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-per-config --no-cpu > gpurun_out/r02c_bench_e2efirst.json 2> gpurun_out/r02c_bench_e2efirst.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02c_ref.json 2> gpurun_out/r02c_ref.err
