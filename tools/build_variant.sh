#!/bin/bash
# Experiment builds: recompile some translation units with extra defines and link them with the
# in-tree objects into paper_0901_1413_b200/libslicegemm_NAME.so (for tools/ab_libs.sh).
#   usage: bash tools/build_variant.sh NAME "-DSG_X_...=1" sg_m4rm_f5 [sg_m4rm_f7 ...]
cd "$(dirname "$0")/../paper_0901_1413_b200/csrc" || exit 1
NAME=$1; DEFS=$2; shift 2
mkdir -p build_$NAME
OBJS=""
for o in build/*.o; do
  b=$(basename $o .o); use=$o
  for t in "$@"; do
    if [ "$t" = "$b" ]; then
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v $DEFS \
          -c $b.cu -o build_$NAME/$b.o > build_$NAME/$b.ptxas.log 2>&1 || { cat build_$NAME/$b.ptxas.log; exit 1; }
      use=build_$NAME/$b.o
    fi
  done
  OBJS="$OBJS $use"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libslicegemm_$NAME.so $OBJS && echo built libslicegemm_$NAME.so
