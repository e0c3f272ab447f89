"""BASELINE configs[3] crypto rollout at full length: 4096 envs, 480,000 one-second
steps (one episode), Q-net 103-128-128-3, epsilon-greedy 0.005 (Philox).

    python scripts/prof_crypto.py [N] [T] [calls]

Prints env-steps/s and the time per lockstep step (all envs advance one step).
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import market  # noqa: E402
from synth import policy as spol  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = int(sys.argv[2]) if len(sys.argv) > 2 else 480000
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 10
t0 = time.time()
rows = market.crypto_market(T, seed=41)
gen_s = time.time() - t0
cfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=T + 1,
                     episode_len=T, reward_scale=1.0, cost_rate=0.0, epsilon=0.005, seed=43)
env = fin.fin_env_create(cfg, rows)
pol = fin.fin_policy_create(fin.FIN_Q_ARGMAX, spol.kaiming_bf16(spol.CRYPTO_DIMS, 4))
Tc = T // calls
rew = torch.zeros((Tc, N), dtype=torch.float32, device="cuda")
done = torch.zeros((Tc, N), dtype=torch.uint8, device="cuda")
agg = torch.zeros(8, dtype=torch.float64, device="cuda")
tr = fin.make_traj(reward=rew, done=done, agg=agg)
nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 43)
# warm-up on a throwaway handle of the same shape (the timed handle starts at step 0)
wenv = fin.fin_env_create(cfg, rows)
fin.fin_rollout(wenv, [pol], min(Tc, 2000), nz, fin.make_traj(reward=rew[:min(Tc, 2000)], done=done[:min(Tc, 2000)]))
torch.cuda.synchronize()
del wenv
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for c in range(calls):
    fin.fin_rollout(env, [pol], Tc, nz, tr)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b)
steps = Tc * calls
print(json.dumps({"workload": "C3 crypto, single asset, 10-level LOB, 101 factors", "envs": N, "steps": steps,
                  "calls": calls, "ms": ms, "env_steps_per_s": N * steps / (ms / 1e3),
                  "us_per_lockstep_step": 1e3 * ms / steps, "market_gen_s": gen_s,
                  "episodes_done": int(done.sum().item())}))
