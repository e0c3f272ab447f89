"""The HBM-bound kernels of bench.py (K1 step at 2^22 envs, K4 replay, K6 metrics), alone."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402

r = bench.hbm_kernels(fin, torch)
for k, v in r.items():
    print(k, {x: v[x] for x in ("ms", "env_steps_per_s", "achieved_gbs", "frac")})
print(json.dumps(r))
