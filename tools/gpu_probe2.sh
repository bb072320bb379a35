#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
./tools/lds_random_probe > gpurun_out/lds_random.jsonl 2>&1; cat gpurun_out/lds_random.jsonl
python tools/prof_one.py --config 4 --m 8192 --reps 2 --rt 16 --threads 256 --pipe 1 --splits 1 > gpurun_out/p3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/p3_f3_rt16_pipe1 python tools/prof_one.py --config 4 --m 8192 --reps 2 --rt 16 --threads 256 --pipe 1 --splits 1 > gpurun_out/p3_ncu.log 2>&1
tail -2 gpurun_out/p3_ncu.log
python tools/prof_one.py --config 3 --m 4096 --reps 2 --rt 8 --threads 256 --pipe 0 --splits 1 > gpurun_out/p4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/p4_f7_rt8 python tools/prof_one.py --config 3 --m 4096 --reps 2 --rt 8 --threads 256 --pipe 0 --splits 1 > gpurun_out/p4_ncu.log 2>&1
tail -2 gpurun_out/p4_ncu.log
