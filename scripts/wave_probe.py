"""Throughput of the fused C1 rollout vs env count (T = 256): exposes wave quantisation
of the one-tile-per-CTA grid (tiles / (2 CTAs x 148 SMs))."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import policy as spol  # noqa: E402

pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
flush = bench.L2Flush(torch)
res = {}
for N in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else
                           "18944,37888,47360,56832,65536,75776".split(","))]:
    env = bench.make_env(fin, N, 0)
    times, _ = bench.time_rollouts(fin, torch, env, pol, N, 256, 5, 3, flush)
    ms = statistics.median(times)
    res[N] = {"tiles": (N + 127) // 128, "ms": ms, "env_steps_per_s": N * 256 / (ms / 1e3)}
    print(N, res[N], flush=True)
    del env
print(json.dumps(res))
