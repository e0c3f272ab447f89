"""Small-N A/B of the pre-drawn rollout noise (DESIGN.md 4.3 "small N"): the C1 fused rollout
(single PPO policy, Philox noise) with FIN_PREGEN=0 (in-kernel draws), 1 (the normals drawn up
front by k_pregen_noise, then read as supplied noise) and 2 (streamed by k_stream_noise on the
idle SMs while the rollout runs) over a sweep of N x T.
Medians of 20 CUDA-event timed calls (pre-draw kernel included), alternated twice.

    python scripts/pregen_ab.py
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


def run(N, T, pre):
    os.environ["FIN_PREGEN"] = pre
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
    c = fin.fin_env_counters(env)
    fin.fin_env_destroy(env)
    return statistics.median(ts), c["pregen_rollouts"]


for N, T in ((64, 256), (2048, 30), (2048, 256), (4096, 256), (8192, 256), (12288, 256), (16384, 256),
             (16384, 30)):
    out = {}
    for rep in range(2):
        for pre in ("0", "1", "2", "3"):
            ms, npre = run(N, T, pre)
            out.setdefault(pre, []).append(ms)
    m0, m1, m2, m3 = min(out["0"]), min(out["1"]), min(out["2"]), min(out["3"])
    print(f"N={N:6d} T={T:4d} in-kernel {m0:.4f} ms ({N * T / m0 * 1e3:.3e}/s)  pre-drawn {m1:.4f} ms "
          f"({m0 / m1 - 1:+.1%})  streamed {m2:.4f} ms ({N * T / m2 * 1e3:.3e}/s, {m0 / m2 - 1:+.1%})  producer-first {m0 / m3 - 1:+.1%}", flush=True)
