"""One fused C1 rollout of N envs x T steps (after one warm-up call) -- for ncu captures.

    python scripts/one_rollout.py N [T]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import policy as spol  # noqa: E402

N = int(sys.argv[1])
T = int(sys.argv[2]) if len(sys.argv) > 2 else 256
pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
env = bench.make_env(fin, N, 0)
z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
traj = fin.make_traj(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8), agg=z(8, torch.float64))
noise = fin.make_noise(fin.FIN_NOISE_PHILOX, 1234)
for _ in range(2):
    fin.fin_rollout(env, [pol], T, noise, traj)
torch.cuda.synchronize()
print("ok", N, T)
print(fin.fin_env_counters(env))
