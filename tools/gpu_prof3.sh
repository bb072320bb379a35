#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/prof_one.py --config 1 --reps 2 > gpurun_out/p5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/p5_f5 python tools/prof_one.py --config 1 --reps 2 > gpurun_out/p5_ncu.log 2>&1
cat gpurun_out/p5_plain.log; tail -1 gpurun_out/p5_ncu.log
python tools/prof_one.py --config 3 --m 4096 --reps 2 > gpurun_out/p6_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/p6_f7 python tools/prof_one.py --config 3 --m 4096 --reps 2 > gpurun_out/p6_ncu.log 2>&1
cat gpurun_out/p6_plain.log; tail -1 gpurun_out/p6_ncu.log
