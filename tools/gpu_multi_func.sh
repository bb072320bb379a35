#!/bin/bash
# functional check of bench.py's N > 1 path on a one-GPU box (2 ranks on cuda:0, gloo collectives)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export SG_BENCH_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-per-config > gpurun_out/multi_head.json 2> gpurun_out/multi_head.err
echo "head rc=$?"; head -c 1500 gpurun_out/multi_head.json; tail -5 gpurun_out/multi_head.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-per-config --config 3 > gpurun_out/multi_f7.json 2> gpurun_out/multi_f7.err
echo "f7 strong rc=$?"; head -c 800 gpurun_out/multi_f7.json; tail -5 gpurun_out/multi_f7.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/multi_ref.json 2> gpurun_out/multi_ref.err
echo "ref rc=$?"; head -c 600 gpurun_out/multi_ref.json; tail -3 gpurun_out/multi_ref.err
