"""Small runs of every kernel of libfinenv.so, for compute-sanitizer (one tool per call):

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_run.py [part ...]

Parts (default: all): k1 k4 k3 ens paper crypto vote k6 market gae kl probe chunk.  C0-sized
envs except ``chunk``, which needs more tiles than resident CTAs (the
dynamic chunk schedule) and runs 38,400 envs for 3 steps.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_10709_b200 import fin  # noqa: E402
from synth import inputs, market  # noqa: E402
from synth import policy as spol  # noqa: E402

z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
parts = sys.argv[1:] or ["k1", "k4", "k3", "ens", "paper", "crypto", "vote", "k6", "market", "gae", "kl", "probe",
                         "chunk"]


def c1_env(N, T_ep=5, **kw):
    m = market.stock_c1(rows=80)
    cfg = fin.env_config(num_envs=N, num_assets=30, num_indicators=8, num_rows=80, episode_len=T_ep, num_windows=10,
                         **kw)
    return fin.fin_env_create(cfg, m.market)


def run(name):
    if name == "k1":
        mk = market.stock_c0()
        cfg = fin.env_config(num_envs=8, num_assets=4, num_indicators=4, num_rows=mk.rows, episode_len=64)
        env = fin.fin_env_create(cfg, mk.market)
        acts = torch.from_numpy(inputs.stock_actions(8, 8, 4, seed=12)).cuda()
        for t in range(8):
            fin.fin_env_step(env, acts[t].contiguous(), fin.make_traj(reward=z(8, torch.float32), done=z(8, torch.uint8)))
        env2 = c1_env(300)
        fin.fin_env_step(env2, z((300, 30), torch.int16) + 7, fin.make_traj(reward=z(300, torch.float32)))
    elif name == "k4":
        env = c1_env(300)
        T = 12
        acts = torch.from_numpy(inputs.stock_actions(T, 300, 30, seed=3)).cuda()
        fin.fin_rollout_actions(env, acts, T, fin.make_traj(reward=z((T, 300), torch.float32),
                                                            ep_metrics=z((3, 300, 3), torch.float64),
                                                            ep_count=z(300, torch.int32), agg=z(8, torch.float64)))
    elif name in ("k3", "paper", "ens"):
        dims = spol.STOCK_PAPER_DIMS if name == "paper" else spol.STOCK_DIMS
        kinds = [fin.FIN_PPO_GAUSS, fin.FIN_SAC_SQUASH, fin.FIN_DDPG_OU] if name == "ens" else [fin.FIN_PPO_GAUSS]
        pols = [fin.fin_policy_create(k, spol.kaiming_bf16(dims, 1 + j)) for j, k in enumerate(kinds)]
        env = c1_env(300)
        T = 7
        fin.fin_rollout(env, pols, T, fin.make_noise(fin.FIN_NOISE_PHILOX, 5),
                        fin.make_traj(reward=z((T, 300), torch.float32), done=z((T, 300), torch.uint8),
                                      agg=z(8, torch.float64)))
        fin.fin_ensemble_act(env, pols, z((300, 30), torch.int16), z((300, 30), torch.float32))
    elif name == "chunk":
        pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
        N, T = 38400, 3
        env = c1_env(N)
        fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_PHILOX, 5),
                        fin.make_traj(reward=z((T, N), torch.float32), agg=z(8, torch.float64)))
        print(fin.fin_env_counters(env))
    elif name in ("crypto", "vote"):
        T, N = 40, 200
        rows = market.crypto_market(T, seed=41)
        cfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=T + 1,
                             episode_len=T, reward_scale=1.0, cost_rate=0.0, epsilon=0.005, seed=43)
        env = fin.fin_env_create(cfg, rows)
        kinds = [fin.FIN_Q_ARGMAX, fin.FIN_Q_ARGMAX, fin.FIN_Q_DUELING] if name == "vote" else [fin.FIN_Q_ARGMAX]
        pols = []
        for j, k in enumerate(kinds):
            d = spol.CRYPTO_DIMS if k == fin.FIN_Q_ARGMAX else tuple(spol.CRYPTO_DIMS[:-1]) + (4,)
            pols.append(fin.fin_policy_create(k, spol.kaiming_bf16(d, 4 + j)))
        fin.fin_rollout(env, pols, T, fin.make_noise(fin.FIN_NOISE_PHILOX, 43),
                        fin.make_traj(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8),
                                      agg=z(8, torch.float64)))
        fin.fin_env_step(env, z((N, 1), torch.int16) + 1, fin.make_traj(reward=z(N, torch.float32)))
    elif name == "k6":
        T, N = 64, 300
        g = torch.Generator(device="cuda").manual_seed(1)
        eq = 1e6 * torch.exp(torch.cumsum(0.01 * torch.randn((T + 1, N), device="cuda", generator=g,
                                                              dtype=torch.float64), 0))
        done = z((T, N), torch.uint8)
        done[29::30] = 1
        fin.fin_episode_metrics(eq, done, 1e6, ep_metrics=z((3, N, 3), torch.float64), ep_count=z(N, torch.int32),
                                agg=z(8, torch.float64))
        N2 = 272   # TMA-staged pass (N % 16 == 0)
        eq2 = eq[:, :N2].contiguous()
        fin.fin_episode_metrics(eq2, done[:, :N2].contiguous(), 1e6, ep_metrics=z((3, N2, 3), torch.float64),
                                ep_count=z(N2, torch.int32), agg=z(8, torch.float64))
    elif name == "market":
        m = market.stock_c0()
        x = np.stack([m.open_all, m.high_all, m.low_all, m.close_all, m.volume_all], axis=1).astype(np.float32)
        D, K = x.shape[0], x.shape[2]
        xd = torch.from_numpy(x).cuda()
        mk = z((D - market.WARMUP_DAYS, 6, K), torch.float32)
        raw = z((4, K, D - market.WARMUP_DAYS), torch.float64)
        fin.fin_market_prepare(xd, market.WARMUP_DAYS, ["macd", "rsi30", "cci30", "sma30"], mk, raw, magnitude=0.01,
                               seed=7)
        rows = z((701, 144), torch.float32)
        fin.fin_crypto_market(700, 43, rows)
    elif name == "gae":
        T, N = 40, 272
        g = torch.Generator(device="cuda").manual_seed(2)
        rew = torch.randn((T, N), device="cuda", generator=g)
        val = torch.randn((T + 1, N), device="cuda", generator=g)
        done = z((T, N), torch.uint8)
        done[9::10] = 1
        adv, ret = torch.empty_like(rew), torch.empty_like(rew)
        fin.fin_gae(rew, val, done, adv, ret, normalise=True)
        fin.fin_gae(rew[:, :250].contiguous(), val[:, :250].contiguous(), done[:, :250].contiguous(),
                    adv[:, :250].contiguous(), ret[:, :250].contiguous())
    elif name == "kl":
        out = torch.tanh(torch.randn((3, 500, 30), device="cuda"))
        fin.fin_kl_diversity(out, z((3, 3), torch.float64))
        fin.fin_kl_diversity(torch.randn((3, 500, 3), device="cuda"), z((3, 3), torch.float64), kind=1)
    elif name == "probe":
        for dims in (spol.STOCK_DIMS, spol.CRYPTO_DIMS):
            kind = fin.FIN_PPO_GAUSS if dims[0] != 103 else fin.FIN_Q_ARGMAX
            pol = fin.fin_policy_create(kind, spol.kaiming_bf16(dims, 0))
            x = torch.zeros((200, dims[0]), dtype=torch.int16, device="cuda")
            fin.fin_mlp_forward(pol, x, z((200, dims[-1]), torch.float32))
    torch.cuda.synchronize()
    print("ok", name, flush=True)


for p in parts:
    run(p)
