"""A/B two builds of libfinenv.so on the crypto rollouts: bitwise output digests and timing.

    python scripts/crypto_ab.py lib_a.so lib_b.so ...

Each library runs in its own process (FIN_LIB_PATH).  Per library: a logged run (network
outputs, hidden activations, rewards, actions) of the C3 Q-net, the paper's 3x128 net and
the 3-member vote at 4,096 envs x 600 steps (digests must agree across libraries), then the
production call (reward + done) timed at 4,096 envs x 48,000 steps, 3 repetitions.
"""
import hashlib
import json
import os
import subprocess
import sys

CHILD = r'''
import hashlib, json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2501_10709_b200 import fin
from synth import market, policy as spol
N, T = 4096, 600
rows = market.crypto_market(48000, seed=41)
cfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=48001,
                     episode_len=48000, reward_scale=1.0, cost_rate=0.0, epsilon=0.005, seed=43)
nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 43)
out = {}
def dig(*ts):
    h = hashlib.sha256()
    for t in ts: h.update(t.cpu().numpy().tobytes())
    return h.hexdigest()[:16]
nets = {"c3": [fin.fin_policy_create(fin.FIN_Q_ARGMAX, spol.kaiming_bf16(spol.CRYPTO_DIMS, 4))],
        "paper": [fin.fin_policy_create(fin.FIN_Q_ARGMAX, spol.kaiming_bf16(spol.CRYPTO_PAPER_DIMS, 4))],
        "vote3": [fin.fin_policy_create(fin.FIN_Q_ARGMAX, spol.kaiming_bf16(spol.CRYPTO_DIMS, 4 + i)) for i in range(3)]}
for name, pols in nets.items():
    env = fin.fin_env_create(cfg, rows)
    M = len(pols)
    rew = torch.zeros((T, N), dtype=torch.float32, device="cuda")
    done = torch.zeros((T, N), dtype=torch.uint8, device="cuda")
    act = torch.zeros((T, N), dtype=torch.int16, device="cuda")
    z = torch.zeros((T, M, N, 3), dtype=torch.float32, device="cuda")
    fin.fin_rollout(env, pols, T, nz, fin.make_traj(reward=rew, done=done, actions=act, mlp_out=z))
    torch.cuda.synchronize()
    out[name] = dig(rew, done, act, z)
env = fin.fin_env_create(cfg, rows)
Tc = 48000
rew = torch.zeros((Tc, N), dtype=torch.float32, device="cuda")
done = torch.zeros((Tc, N), dtype=torch.uint8, device="cuda")
tr = fin.make_traj(reward=rew, done=done)
wenv = fin.fin_env_create(cfg, rows)
fin.fin_rollout(wenv, nets["c3"], 2000, nz, fin.make_traj(reward=rew[:2000], done=done[:2000]))
torch.cuda.synchronize()
us = []
for r in range(3):
    env = fin.fin_env_create(cfg, rows)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fin.fin_rollout(env, nets["c3"], Tc, nz, tr); b.record(); torch.cuda.synchronize()
    us.append(1e3 * a.elapsed_time(b) / Tc)
out["us_per_step"] = us
print("RESULT " + json.dumps(out))
'''

res = {}
for lib in sys.argv[1:]:
    env = dict(os.environ, FIN_LIB_PATH=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    res[lib] = json.loads(line[0][7:]) if line else {"error": p.stderr[-2000:]}
    print(lib, json.dumps(res[lib]), flush=True)
keys = ("c3", "paper", "vote3")
libs = [l for l in res if "error" not in res[l]]
print("bitwise equal:", {k: len({res[l][k] for l in libs}) == 1 for k in keys})
