"""Run pack / unpack once on a 16384 x 32768 F3 matrix (for ncu captures of the HBM-bound kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
print(bench.run_pack_unpack(dev, "f3", 16384, 32768, reps=2))
