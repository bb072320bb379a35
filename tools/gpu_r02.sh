#!/bin/bash
# Round-2 GPU measurement steps (run on the B200 box through gpurun; outputs in gpurun_out/, the
# ones judged are summarized / copied under profiles/).   usage: bash tools/gpu_r02.sh STEP [TAG]
#   probes    TMEM ld/st bandwidth probe, host<->device small-transfer probe (copy engine vs SM)
#   ncu CFG   ncu --set full (+ source) of the M4RM kernel of BASELINE config CFG, raw + SASS CSV
#   small     fused small-product kernels: parity tests, per-CTA phase timeline, bench-style steps
#   grid      bench-style step times of every fused / unfused variant x split count on small shapes
#             (input of tools/fit_calib.py for the fused variants' planner constants)
#   e2e CFG   host-buffer end-to-end probe of config CFG (default pipeline and alternatives)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
STEP=$1; ARG=$2; T=${TAG:-r02}
case $STEP in
probes)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_probe tools/tmem_probe.cu && \
    timeout 120 /tmp/tmem_probe > gpurun_out/${T}_tmem_probe.txt 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/zc_probe tools/zc_probe.cu && \
    timeout 120 /tmp/zc_probe > gpurun_out/${T}_zc_probe.txt 2>&1 ;;
ncu)
  C=${ARG:-1}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o /tmp/${T}_cfg$C \
      python tools/prof_one.py --config $C --reps 2 > gpurun_out/${T}_cfg${C}_ncu.log 2>&1
  ncu -i /tmp/${T}_cfg$C.ncu-rep --page raw --csv > gpurun_out/${T}_ncu_cfg${C}_raw.csv 2>/dev/null
  ncu -i /tmp/${T}_cfg$C.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_ncu_cfg${C}_sass.csv 2>/dev/null ;;
small)
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "fused_small" -x -p no:cacheprovider \
      > gpurun_out/${T}_pytest_fused.txt 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSG_TIMELINE -lcuda -o /tmp/small_timeline \
      tools/small_timeline.cu && timeout 120 /tmp/small_timeline > gpurun_out/${T}_small_timeline.txt 2>&1
  for s in f3:1024:1024:1024 gf4:1024:1024:1024 f5:1024:1024:1024; do
    timeout 300 python tools/step_probe.py --shape $s > gpurun_out/${T}_step_${s%%:*}.txt 2>&1
  done ;;
grid)
  SH=""
  for f in f3 f5 f7 gf4; do for s in 512:512:512 1024:1024:1024 2048:2048:2048 1024:4096:1024 256:2048:2048 \
      2048:1024:2048 4096:512:4096 1024:1024:4096; do SH="$SH,$f:$s"; done; done
  timeout 2400 python tools/step_probe.py --json --grid --steps 10 --shape "${SH#,}" \
      > gpurun_out/${T}_step_grid.jsonl 2> gpurun_out/${T}_step_grid.err ;;
e2e)
  C=${ARG:-1}
  timeout 300 python tools/e2e_probe.py $C > gpurun_out/${T}_e2e_cfg$C.txt 2>&1 ;;
pieces)  # streamed host pipeline: row-piece weight variants (SG_HOST_PIECES), twice each
  for rep in 1 2; do for P in 1,1 1,2,1 1,3 1,2,2,1 1,1,1,1 2,3,1 1,2,1,1 1,4,2,1; do
    SG_HOST_PIECES=$P timeout 120 python tools/e2e_probe.py 1 2>&1 | sed "s/^/pieces=$P /" >> gpurun_out/${T}_e2e_pieces.txt
  done; done ;;
launches)  # ncu launch list of the bench command (per-kernel durations, cold-cache, serialised)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/${T}_launches_bench.json 2>&1 ;;
trace)  # event trace of one streamed host call of config ARG (default 1), three processes
  for i in 1 2 3; do TRACE=1 timeout 120 python tools/e2e_probe.py ${ARG:-1} >> gpurun_out/${T}_e2e_trace.txt 2>&1; done ;;
suite)
  timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.txt 2>&1
  echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.txt ;;
bench)
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
  echo "bench exit $?" >> gpurun_out/${T}_bench.err ;;
esac
