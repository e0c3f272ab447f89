"""One DDPG and one SAC update at B = 65,536 (after warm-up) -- for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "ddpg"
print(bench.ac_update(fin, torch, kind, 65536))
