#!/bin/bash
# ncu captures of the M4RM kernel for one config: launch list + one --set full capture.
# usage: bash tools/gpu_prof.sh CONFIG TAG [extra prof_one args]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=$1; TAG=$2; shift 2
mkdir -p gpurun_out
python tools/prof_one.py --config $CFG --reps 2 "$@" > gpurun_out/prof_${TAG}_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/prof_${TAG}_plain.log; exit 1; }
cat gpurun_out/prof_${TAG}_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_${TAG}_launches.csv python tools/prof_one.py --config $CFG --reps 2 "$@" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG} python tools/prof_one.py --config $CFG --reps 2 "$@" > gpurun_out/prof_${TAG}_ncu.log 2>&1
tail -3 gpurun_out/prof_${TAG}_ncu.log
ls -la gpurun_out/
