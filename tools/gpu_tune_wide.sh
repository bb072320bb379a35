#!/bin/bash
# wide tune sweep for the planner fit: BASELINE configs + sharded per-rank shapes + mid-size and
# skinny shapes for every calibrated field (profiles/<tag>_tune_wide.jsonl)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r01}
SH="f3:4096:32768:32768,f7:2048:8192:16384,gf4:4096:8192:8192,f5:2048:4096:4096"
SH="$SH,f3:2048:2048:2048,f3:8192:1024:8192,f3:512:8192:4096,f3:16384:4096:1024"
SH="$SH,f5:1000:1000:1000,f5:16384:1024:512,f5:2048:8192:2048,f5:8192:2048:8192"
SH="$SH,f7:3000:5000:2000,f7:1024:4096:4096,f7:8192:1024:8192"
SH="$SH,gf4:2500:2500:2500,gf4:16384:2048:4096,gf4:1024:16384:1024"
timeout 2400 python tools/tune.py --configs 0,1,2,3 --shapes $SH --reps 2 > gpurun_out/${TAG}_tune_wide.jsonl 2> gpurun_out/${TAG}_tune_wide.err
echo "tune rc=$?"
python - "$TAG" << 'PY'
import json, sys
tag = sys.argv[1]
for l in open(f"gpurun_out/{tag}_tune_wide.jsonl"):
    r = json.loads(l)
    if "BEST" in r and r["BEST"]:
        print(r["config"], "auto/best %.2f" % (r["auto_plan"]["ms"] / r["BEST"]["ms"]))
PY
