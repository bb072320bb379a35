"""Pack / unpack HBM throughput of the loaded library build (bench.run_pack_unpack), for A/B via
SG_LIB_PATH.   python tools/pack_ab.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
for field, m, n in (("f3", 16384, 32768), ("f5", 16384, 16384), ("gf4", 8192, 8192), ("f7", 4099, 10007), ("f7", 4099, 10008),
                    ("f5", 5000, 10004), ("f3", 3000, 1000)):
    r = bench.run_pack_unpack(dev, field=field, m=m, n=n, reps=9)
    print(field, m, n, json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in r.items()
                                   if k in ("pack_ms", "unpack_ms", "pack_gbps", "unpack_gbps", "pack_frac", "unpack_frac")}))
