"""Needs a build with the timeline compiled in:
    FIN_NVCC_FLAGS=-DFIN_TRACE python -m paper_2501_10709_b200.build --force
Print the block-0 clock64 timeline of a fused rollout (fin_debug_trace), in cycles
relative to the start of each step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import market  # noqa: E402
from synth import policy as spol  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
m = market.stock_c1(rows=1008)
cfg = fin.env_config(num_envs=N, num_assets=30, num_indicators=8, num_rows=1008, episode_len=30, num_windows=195)
env = fin.fin_env_create(cfg, m.market)
pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
rew = torch.zeros((T, N), dtype=torch.float32, device="cuda")
tr = fin.make_traj(reward=rew)
nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 7)
fin.fin_rollout(env, [pol], T, nz, tr)
buf = torch.zeros((3 * T, 32), dtype=torch.int64, device="cuda")
fin.fin_debug_trace(buf)
fin.fin_rollout(env, [pol], T, nz, tr)
torch.cuda.synchronize()
fin.fin_debug_trace(None)
b = buf.cpu().numpy().astype(np.int64)
names = {0: "step", 23: "stg:d", 24: "stg:uni", 25: "stg:done", 1: "obs_done", 9: "mma:a1", 10: "mma:i1",
         2: "d1", 3: "epi1", 11: "mma:a2", 12: "mma:i2", 4: "d2", 5: "epi2", 13: "mma:a3", 14: "mma:i3", 6: "d3",
         16: "philox0", 7: "consume", 26: "w1rdy", 27: "w2rdy", 28: "w3rdy", 29: "w2last", 30: "p:l1", 31: "p:l3", 17: "fs:start", 19: "fs:body", 20: "fs:tx", 21: "fs:metric", 8: "env_done"}
for t in range(T):
    d = b[t] - b[t, 0]
    order = sorted((int(d[i]), n) for i, n in names.items() if b[t, i] != 0)
    print(f"t={t}: " + " ".join(f"{n}={v}" for v, n in order))

# per-stage detail: MMA warp after each stage's w_full wait (m) / producer after each w_empty wait (p)
for t in range(T):
    d = b[T + t] - b[t, 0]
    print(f"t={t} stages: " + " ".join(f"m{s}={int(d[s])}" for s in range(16) if b[T + t, s] != 0))
    print(f"t={t} produce: " + " ".join(f"p{s}={int(d[16 + s])}" for s in range(16) if b[T + t, 16 + s] != 0))
    d = b[2 * T + t] - b[t, 0]
    print(f"t={t} mma before-wait/after-issue: " + " ".join(f"s{s}={int(d[s])}/{int(d[16 + s])}" for s in range(16) if b[2 * T + t, s] != 0))
