"""Debug: streamed noise (FIN_PREGEN=2) vs in-kernel draws on a small rollout; prints the call
time, the sticky flags and where the actions differ."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import market  # noqa: E402
from synth import policy as spol  # noqa: E402

N, T = int(sys.argv[1]) if len(sys.argv) > 1 else 260, int(sys.argv[2]) if len(sys.argv) > 2 else 8
m = market.stock_c1(rows=100)
pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
res = {}
for mode in ("0", "1", "2", "2"):
    os.environ["FIN_PREGEN"] = mode
    cfg = fin.env_config(task=fin.FIN_STOCK, num_envs=N, num_assets=30, num_indicators=8, num_rows=100, episode_len=5,
                         num_windows=10, window_block=128)
    env = fin.fin_env_create(cfg, m.market)
    a = torch.zeros((T, N, 30), dtype=torch.int16, device="cuda")
    torch.cuda.synchronize()
    t0 = time.time()
    fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_PHILOX, 1234), fin.make_traj(actions=a))
    torch.cuda.synchronize()
    dt = time.time() - t0
    try:
        fl = fin.fin_env_check(env)
    except Exception as ex:  # noqa: BLE001
        fl = str(ex)
    c = fin.fin_env_counters(env)
    r = a.cpu().numpy()
    if mode != "0":
        d = np.argwhere(r != res["0"])
        print(f"mode {mode}: {dt * 1e3:.1f} ms flags {fl} counters {c} differing {len(d)} first {d[:5].tolist()}")
    else:
        res["0"] = r
        print(f"mode 0: {dt * 1e3:.1f} ms flags {fl}")
    fin.fin_env_destroy(env)
