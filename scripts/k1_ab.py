"""K1 (fin_env_step, N = 2^22) and K4 rates of the library FIN_LIB_PATH points to (A/B runs).

    FIN_LIB_PATH=... python scripts/k1_ab.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402

r = bench.hbm_kernels(fin, torch)
print(os.path.basename(fin.LIB_PATH), round(r["step_kernel_hbm"]["achieved_gbs"]), round(r["replay_kernel_hbm"]["achieved_gbs"]))
