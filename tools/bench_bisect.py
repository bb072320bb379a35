"""Which part of bench.py's flow slows the e2e host pipeline that follows it?  usage:
python tools/bench_bisect.py [probe] [config] -> the e2e line after the selected parts"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_0901_1413_b200 import m4rm as M  # noqa: E402


class Args:
    steps, warmup = 10, 3


parts = sys.argv[1:]
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
peaks = {"lop3_per_clk_per_sm": 64.0, "lds_bytes_per_clk_per_sm": 128.0, "clock_mhz_for_peak": 1965.0,
         "clock_note": ""}
if "probe" in parts:
    M.probe_peaks(0)
if "config" in parts:
    bench.run_config(bench.CONFIGS[bench.HEADLINE], Args, 1, 0, dev, peaks, e2e=False)
e = bench.e2e_for(bench.CONFIGS[bench.HEADLINE], Args, 1, 0, dev)
print(parts, "e2e %.3f ms" % e["ms_per_step"], flush=True)
