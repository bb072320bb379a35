#!/bin/bash
# e2e variants + the GPU test suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
O=gpurun_out/r02b_e2e.txt
: > $O
TRACE=1 timeout 300 python tools/e2e_probe.py 1 >> $O 2>&1
VARIANT=stream0 SG_HOST_STREAM=0 timeout 300 python tools/e2e_probe.py 1 >> $O 2>&1
for c in 1 2 4; do VARIANT=chunks$c SG_HOST_CHUNKS=$c timeout 300 python tools/e2e_probe.py 1 >> $O 2>&1; done
timeout 300 python tools/e2e_probe.py 1 >> $O 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r02b_pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r02b_pytest_gpu.txt
