#!/bin/bash
# two ncu --set full captures of the M4RM kernel (config $1, m=$2) for pipe=0 and pipe=1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for P in 0 1; do
  python tools/prof_one.py --config $1 --m $2 --reps 2 --pipe $P --rt $3 --splits $4 > gpurun_out/p2_${P}_plain.log 2>&1 || { cat gpurun_out/p2_${P}_plain.log; exit 1; }
  cat gpurun_out/p2_${P}_plain.log
  ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/p2_cfg$1_pipe$P python tools/prof_one.py --config $1 --m $2 --reps 2 --pipe $P --rt $3 --splits $4 > gpurun_out/p2_${P}_ncu.log 2>&1
  tail -2 gpurun_out/p2_${P}_ncu.log
done
