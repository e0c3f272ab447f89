"""Per-tile cost of the fused C1 rollout (debug FIN_SEG_PROF timeline): N envs, one tile per
CTA when N <= 148 x 128, for several window bases."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_10709_b200 import fin  # noqa: E402
from synth import market  # noqa: E402
from synth import policy as spol  # noqa: E402

N, T = int(sys.argv[1]), 256
out = sys.argv[2]
m = market.stock_c1(rows=1008)
pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
res = []
for base in (0, 48, 96, 144):
    cfg = fin.env_config(num_envs=N, num_assets=30, num_indicators=8, num_rows=1008, episode_len=30, window_stride=5,
                         num_windows=195, window_block=128, window_base=base, seed=23)
    env = fin.fin_env_create(cfg, m.market)
    tr = fin.make_traj(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8))
    nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 1234)
    fin.fin_rollout(env, [pol], T, nz, tr)
    os.environ["FIN_SEG_PROF"] = "/tmp/prof.bin"
    fin.fin_rollout(env, [pol], T, nz, tr)
    del os.environ["FIN_SEG_PROF"]
    a = np.fromfile("/tmp/prof.bin", dtype=np.uint64).reshape(-1, 16).astype(np.int64)
    ntile = (N + 127) // 128
    dt = (a[:ntile, 2] - a[:ntile, 1]) / 1e3 / T
    for j in range(ntile):
        res.append((base, j, (base + j) % 195, dt[j], int(a[j, 15])))
np.save(out, np.array(res))
r = np.array(res)
print("us/step: min %.2f max %.2f mean %.2f" % (r[:, 3].min(), r[:, 3].max(), r[:, 3].mean()))
