"""Small fused-rollout run for ncu (one launch of interest after warm-up).

    python scripts/prof_rollout.py [N] [T] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import market  # noqa: E402
from synth import policy as spol  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
m = market.stock_c1(rows=1008)
cfg = fin.env_config(num_envs=N, num_assets=30, num_indicators=8, num_rows=1008, episode_len=30, num_windows=195)
env = fin.fin_env_create(cfg, m.market)
pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
rew = torch.zeros((T, N), dtype=torch.float32, device="cuda")
done = torch.zeros((T, N), dtype=torch.uint8, device="cuda")
agg = torch.zeros(8, dtype=torch.float64, device="cuda")
tr = fin.make_traj(reward=rew, done=done, agg=agg)
nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 7)
for _ in range(reps):
    fin.fin_rollout(env, [pol], T, nz, tr)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
fin.fin_rollout(env, [pol], T, nz, tr)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e)
print(f"N={N} T={T}: {ms:.3f} ms  {N*T/ms/1e3:.3e} env-steps/s  {ms*1e3/T:.2f} us/step")
