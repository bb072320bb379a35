cd ${GRAFT_REPO_ROOT:-/root/repo}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tmem_accumulator or fuzz or streamk_forced" -p no:cacheprovider > gpurun_out/r02bq_pytest_tm.txt 2>&1; tail -3 gpurun_out/r02bq_pytest_tm.txt
for f in gf8 z8; do timeout 300 python tools/step_probe.py --steps 10 --plans "16,-1,6,256;8,-1,2,256" --shape $f:8192:8192:8192,$f:4096:4096:4096,$f:16384:8192:16384 2>&1 | grep -v "^(1, \|^(2, \|^(4, " | sed "s/^/$f /"; done > gpurun_out/r02bq_step_tm_fields.txt 2>&1
for f in z4 f2; do timeout 300 python tools/step_probe.py --steps 10 --plans "32,-1,6,256;16,-1,2,256" --shape $f:8192:8192:8192,$f:4096:4096:4096,$f:16384:16384:16384 2>&1 | grep -v "^(1, \|^(2, \|^(4, " | sed "s/^/$f /"; done >> gpurun_out/r02bq_step_tm_fields.txt 2>&1
cut -c1-150 gpurun_out/r02bq_step_tm_fields.txt
