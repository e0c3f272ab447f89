"""Diagnostic: fused-rollout network outputs vs the K7 probe on the oracle's observation."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import mlp as omlp  # noqa: E402
from oracle import rollout as orol  # noqa: E402
from oracle import stock as ostock  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import inputs, market  # noqa: E402
from synth import policy as spol  # noqa: E402

m = market.stock_c1(rows=60)
N, T, K = 130, 3, 30
ocfg = ostock.StockEnvConfig(num_envs=N, num_assets=K, num_indicators=8, num_rows=60, episode_len=5, num_windows=8)
fcfg = fin.env_config(num_envs=N, num_assets=K, num_indicators=8, num_rows=60, episode_len=5, num_windows=8)
env = fin.fin_env_create(fcfg, m.market)
layers = spol.kaiming_bf16(spol.STOCK_DIMS, 0)
pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, layers)
noise = inputs.supplied_noise(T, 1, N, K, seed=23)
z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
logs = dict(actions=z((T, N, K), torch.int16), mlp_out=z((T, 1, N, K), torch.float32))
fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_SUPPLIED, 0, torch.from_numpy(noise).cuda()),
                fin.make_traj(**logs))
torch.cuda.synchronize()
g = {k: v.cpu().numpy() for k, v in logs.items()}
st = ostock.reset(ocfg)
L64 = omlp.layers_f64(layers)
for t in range(T):
    X = orol.stock_obs_batch(ocfg, st, m.market)
    ref = omlp.forward(L64, X)
    xb = spol.f64_to_bf16_bits(X).view(np.int16)
    zp = z((N, K), torch.float32)
    fin.fin_mlp_forward(pol, torch.from_numpy(xb).cuda(), zp)
    probe = zp.cpu().numpy().astype(np.float64)
    got = g["mlp_out"][t, 0].astype(np.float64)
    print(f"t={t} |probe-ref| max {np.abs(probe-ref).max():.3e}  |rollout-ref| max {np.abs(got-ref).max():.3e}"
          f"  |rollout-probe| max {np.abs(got-probe).max():.3e}  ref rms {np.sqrt((ref**2).mean()):.3e}")
    bad = np.argwhere(np.abs(got - probe) > 1e-3)
    print("  bad (env,k) first:", bad[:10].tolist(), "count", len(bad))
    if len(bad):
        i = bad[0][0]
        print("  got", got[i, :6], "\n  probe", probe[i, :6])
    ostock.step(ocfg, st, m.market, g["actions"][t])
