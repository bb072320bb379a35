#!/bin/bash
# Profile set for profiles/ (one call on the B200): bench line + reference arm, the ncu launch list
# of the bench command, `ncu --set full` of the M4RM kernel for every BASELINE config (exported to
# CSV on the box: raw metrics + details page), and the launch list of one streamed e2e call.
# usage: bash tools/gpu_profiles_full.sh TAG      (then: tools/ncu_summary.py, pipes/traffic_from_ncu.py)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference_arm.json 2> /dev/null
echo "reference arm rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_launches_bench.json 2>&1
echo "launch list rc=$?"
for C in 1 2 3 4 0; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o /tmp/${TAG}_cfg$C \
      python tools/prof_one.py --config $C --reps 2 > gpurun_out/${TAG}_cfg${C}_ncu.log 2>&1
  echo "cfg$C full rc=$?"
  ncu -i /tmp/${TAG}_cfg$C.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_cfg${C}_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_cfg$C.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_cfg${C}_details.csv 2>/dev/null
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_e2e_launches.csv \
    python tools/e2e_probe.py 1 > gpurun_out/${TAG}_e2e_launches.log 2>&1
echo "e2e launch list rc=$?"
ls -la gpurun_out | grep ${TAG}
