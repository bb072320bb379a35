#!/bin/bash
# Evidence for profiles/: plain bench, ncu launch list of the same bench command, and one
# `ncu --set full` capture of the M4RM kernel for the headline config (1) and for config 4.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r01}
python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_launches_bench.json 2>&1
echo "launch list rc=$?"
python tools/prof_one.py --config 1 --reps 2 > gpurun_out/${TAG}_cfg1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/${TAG}_cfg1_m4rm \
    python tools/prof_one.py --config 1 --reps 2 > gpurun_out/${TAG}_cfg1_ncu.log 2>&1
echo "cfg1 full rc=$?"
python tools/prof_one.py --config 4 --reps 1 > gpurun_out/${TAG}_cfg4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:m4rm_kernel -s 1 -c 1 -o gpurun_out/${TAG}_cfg4_m4rm \
    python tools/prof_one.py --config 4 --reps 1 > gpurun_out/${TAG}_cfg4_ncu.log 2>&1
echo "cfg4 full rc=$?"
ls -la gpurun_out | tail -12
