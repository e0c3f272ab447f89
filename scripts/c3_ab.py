"""C3 crypto rollout rate (bench.crypto_c3) of the library FIN_LIB_PATH points to (A/B runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402

r = bench.crypto_c3(fin, torch)
print(os.path.basename(fin.LIB_PATH), round(r["us_per_lockstep_step"], 4))
