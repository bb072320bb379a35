#!/bin/bash
# A/B of two builds of the library on bench-style step times (tools/step_probe.py), alternating
# processes.   usage: bash tools/ab_libs.sh TAG "shape,shape,..." [ROUNDS] ["lib names"]
# A = paper_0901_1413_b200/libslicegemm_base.so (a build of the code before the change),
# B = the in-tree build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=$1; SH=$2; N=${3:-3}; LIBS=${4:-"base b200"}
OUT=gpurun_out/${T}_ab.txt
: > $OUT
for i in $(seq $N); do
  for L in $LIBS; do
    echo "== round $i lib $L" >> $OUT
    SG_LIB_PATH=$PWD/paper_0901_1413_b200/libslicegemm_$L.so timeout 600 python tools/step_probe.py \
        --shape "$SH" --plans "0,0,-1,0" --steps 20 2>&1 | grep -v "^$" >> $OUT
  done
done
cat $OUT
