#!/bin/bash
# A/B of the stream-K hybrid (whole-tile waves + a stream-K tail) against pure stream-K ranges
# (SG_STREAMK_HYBRID=0), bench-style steps, alternating processes; then ncu captures for the
# DRAM traffic.   usage: bash tools/hybrid_ab.sh TAG
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; T=${1:-r02bt}
SH="f3:32768:32768:32768,f3:16384:32768:32768,f7:16384:8192:16384,gf4:16384:16384:16384,f5:16384:16384:16384"
: > gpurun_out/${T}_hybrid_ab.txt
for i in 1 2; do for H in 1 0; do
  echo "== round $i SG_STREAMK_HYBRID=$H" >> gpurun_out/${T}_hybrid_ab.txt
  SG_STREAMK_HYBRID=$H timeout 900 python tools/step_probe.py --steps 6 --plans "0,-1,-1,0" --shape $SH 2>&1 | grep "^(0, " | cut -c1-150 >> gpurun_out/${T}_hybrid_ab.txt
done; done
cat gpurun_out/${T}_hybrid_ab.txt
