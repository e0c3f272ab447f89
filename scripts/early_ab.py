"""(run once per library, FIN_LIB_PATH) Small-N A/B of the noise placement in the STREAM kernel; derived from split_ab.py: the column-split epilogues: the C1 fused rollout (single PPO
policy, Philox noise, default small-N noise mode) with FIN_SPLIT=0 (one env warpgroup) vs the
default (the hidden epilogues split over two warpgroups), and the in-kernel-noise baseline
(FIN_PREGEN=0).  Best of two medians of 20 CUDA-event timed calls.

    python scripts/split_ab.py
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import policy as spol  # noqa: E402

pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
VARIANTS = {"base": {"FIN_PREGEN": "0", "FIN_SPLIT": "0"}, "default": {}, "mode4": {"FIN_PREGEN": "4"}, "mode2": {"FIN_PREGEN": "2"}}


def run(N, T, env_vars):
    for k in ("FIN_PREGEN", "FIN_SPLIT"):
        os.environ.pop(k, None)
    os.environ.update(env_vars)
    env = bench.make_env(fin, N, 0)
    nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 3)
    tr = fin.make_traj(reward=torch.zeros((T, N), device="cuda"),
                       done=torch.zeros((T, N), dtype=torch.uint8, device="cuda"))
    for _ in range(3):
        fin.fin_rollout(env, [pol], T, nz, tr)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fin.fin_rollout(env, [pol], T, nz, tr)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    assert fin.fin_env_check(env) == 0
    fin.fin_env_destroy(env)
    return statistics.median(ts)


for N, T in ((64, 256), (2048, 30), (2048, 256), (8192, 256), (12288, 256), (16384, 256)):
    out = {}
    for rep in range(2):
        for name, ev in VARIANTS.items():
            out.setdefault(name, []).append(run(N, T, ev))
    best = {k: min(v) for k, v in out.items()}
    b0 = best["base"]
    print(f"N={N:6d} T={T:4d} " + "  ".join(f"{k} {v:.4f} ms ({N * T / v * 1e3:.3e}/s, {b0 / v - 1:+.1%})"
                                            for k, v in best.items()), flush=True)
