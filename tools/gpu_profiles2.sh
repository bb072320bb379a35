#!/bin/bash
# ncu --set full captures of the M4RM kernel for BASELINE configs 2 (GF(4) 8192^3) and 3 (F7)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r01}
for C in 2 3 0; do
  python tools/prof_one.py --config $C --reps 2 > gpurun_out/${TAG}_cfg${C}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/${TAG}_cfg${C}_m4rm \
      python tools/prof_one.py --config $C --reps 2 > gpurun_out/${TAG}_cfg${C}_ncu.log 2>&1
  echo "cfg$C full rc=$?"
done
