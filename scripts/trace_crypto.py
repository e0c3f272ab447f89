"""Needs a build with the timeline compiled in:
    FIN_NVCC_FLAGS=-DFIN_TRACE python -m paper_2501_10709_b200.build --force
Block-0 clock64 timeline of the fused crypto rollout (fin_debug_trace), cycles
relative to the start of each step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import market  # noqa: E402
from synth import policy as spol  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rows = market.crypto_market(2000, seed=41)
cfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=2001,
                     episode_len=2000, reward_scale=1.0, cost_rate=0.0, epsilon=0.005, seed=43)
env = fin.fin_env_create(cfg, rows)
pol = fin.fin_policy_create(fin.FIN_Q_ARGMAX, spol.kaiming_bf16(spol.CRYPTO_DIMS, 4))
rew = torch.zeros((T, N), dtype=torch.float32, device="cuda")
tr = fin.make_traj(reward=rew)
nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 7)
fin.fin_rollout(env, [pol], T, nz, tr)
buf = torch.zeros((T, 32), dtype=torch.int64, device="cuda")
fin.fin_debug_trace(buf)
fin.fin_rollout(env, [pol], T, nz, tr)
torch.cuda.synchronize()
fin.fin_debug_trace(None)
b = buf.cpu().numpy().astype(np.int64)
names = {0: "step", 1: "obs_done", 9: "mma:a1", 10: "mma:i1", 2: "d1", 3: "epi1", 11: "mma:a2", 12: "mma:i2",
         4: "d2", 5: "epi2", 13: "mma:a3", 14: "mma:i3", 6: "d3", 7: "consume", 8: "env_done",
         20: "st:wait+bar", 21: "st:red", 22: "st:ring", 27: "st:bcast", 23: "st:prefetch", 24: "st:bar", 25: "kick:bar", 26: "kick:mma"}
for t in range(T):
    d = b[t] - b[t, 0]
    order = sorted((int(d[i]), n) for i, n in names.items() if b[t, i] != 0)
    print(f"t={t}: " + " ".join(f"{n}={v}" for v, n in order))
