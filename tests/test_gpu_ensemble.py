"""GPU parity of the ensemble rules against the oracle.

* fin_member_weights: Sharpe-softmax weights with gating vs
  oracle.policy.softmax_weights on the same statistics.
* Stock weighted ensembles: several PPO / SAC / DDPG members (several
  DDPG members = several OU states), executed action = weighted sum; up to 15 members
  (members 4.. read biases and the factored layer-1 term from L2).  Teacher forced as in
  test_gpu_policy.py.
* validate_and_weight: the validation rollouts' Sharpe ratios and the weights, from
  the oracle's metrics on the replayed validation equity.
* Crypto majority vote: DQN / Double DQN / Dueling DQN members, plurality
  with hold-preferring ties, then epsilon-greedy; 3 members (resident Q-nets) and 9
  members (streamed Q-nets).
"""
import math

import numpy as np
import pytest

from gpu_util import dev, host, needs_gpu, stock_pair, zeros
from oracle import crypto as ocry
from oracle import metrics as omet
from oracle import mlp as omlp
from oracle import policy as opol
from oracle import rollout as orol
from oracle import stock as ostock
from synth import inputs, market
from synth import policy as spol

pytestmark = [pytest.mark.gpu, needs_gpu]


def _fin():
    from paper_2501_10709_b200 import fin
    return fin


# ------------------------------------------------------------------ weights
@pytest.mark.parametrize("M", [1, 3, 15, 30])
def test_member_weights_match_oracle(M):
    import torch
    fin = _fin()
    rng = np.random.default_rng(M)
    for trial in range(20):
        aggs = np.zeros((M, fin.FIN_AGG_LEN))
        aggs[:, fin.FIN_AGG_N_SHARPE] = rng.integers(0, 6, M)
        aggs[:, fin.FIN_AGG_SUM_SHARPE] = rng.normal(0.3, 1.0, M) * aggs[:, fin.FIN_AGG_N_SHARPE]
        thr = float(rng.normal(0.0, 0.6)) if trial % 4 else -math.inf
        tau = float(rng.uniform(0.3, 2.0))
        w, sh = zeros(M, torch.float32), zeros(M, torch.float64)
        fin.fin_member_weights(dev(aggs), w, sh, thr, tau)
        sharpes = [a[fin.FIN_AGG_SUM_SHARPE] / a[fin.FIN_AGG_N_SHARPE] if a[fin.FIN_AGG_N_SHARPE] > 0 else math.nan
                   for a in aggs]
        ref = opol.softmax_weights(sharpes, thr, tau)
        np.testing.assert_allclose(host(w), ref, rtol=1e-6, atol=1e-7)
        np.testing.assert_array_equal(np.isnan(host(sh)), np.isnan(sharpes))
        np.testing.assert_allclose(host(sh)[~np.isnan(sharpes)], np.array(sharpes)[~np.isnan(sharpes)], rtol=1e-15)


# ------------------------------------------------------------------ stock weighted ensemble
def _run_stock(N, T, spec, L, weights=None, rows=150, seed_noise=33, noise_mode=None, **env_kw):
    import torch
    fin = _fin()
    m = market.stock_c1(rows=rows)
    K = 30
    kw = dict(num_envs=N, num_assets=K, num_indicators=8, num_rows=rows, episode_len=L, window_stride=5,
              window_block=128)
    kw.update(env_kw)
    kw["num_windows"] = (rows - 1 - L - kw.get("window_offset", 0)) // 5 + 1
    ocfg, fcfg = stock_pair(**kw)
    env = fin.fin_env_create(fcfg, m.market)
    layers = []
    for s, _, biased in spec:
        L_ = spol.kaiming_bf16(spol.STOCK_DIMS, s)
        layers.append(spol.random_bias(L_, 100 + s) if biased else L_)
    kinds = [k for _, k, _ in spec]
    pols = [fin.fin_policy_create(k, L_) for k, L_ in zip(kinds, layers)]
    M = len(pols)
    noise = inputs.supplied_noise(T, M, N, K, seed=seed_noise)
    E = T // L + 2
    logs = dict(reward=zeros((T, N), torch.float32), done=zeros((T, N), torch.uint8),
                actions=zeros((T, N, K), torch.int16), cash=zeros((T, N), torch.float64),
                hold=zeros((T, N, K), torch.int16), asset=zeros((T, N), torch.float64),
                mlp_out=zeros((T, M, N, K), torch.float32), mlp_hidden=zeros((T, M, N, 2, 256), torch.int16),
                ep_metrics=zeros((E, N, 3), torch.float64), ep_count=zeros(N, torch.int32))
    fin.fin_rollout(env, pols, T, fin.make_noise(fin.FIN_NOISE_SUPPLIED, 0, dev(noise)), fin.make_traj(**logs),
                    member_w=weights)
    g = {k: host(v) for k, v in logs.items()}
    assert fin.fin_env_check(env) == 0
    return g, ocfg, m.market, layers, kinds, noise


def _teacher_forced(g, ocfg, mk, layers, kinds, noise, weights=None, mlp_every=1):
    T, N, K = g["actions"].shape
    o, _ = ostock.run_actions(ocfg, mk, g["actions"])
    assert np.array_equal(g["hold"], o["hold"]) and np.array_equal(g["done"].astype(bool), o["done"])
    assert np.array_equal(g["cash"], o["cash"]) and np.array_equal(g["asset"], o["asset"])
    L64 = [omlp.layers_f64(L_) for L_ in layers]
    st = ostock.reset(ocfg)
    n_ddpg = sum(1 for k in kinds if k == orol.DDPG_OU)
    ou = [[[0.0] * K for _ in range(max(n_ddpg, 1))] for _ in range(N)]
    w = None if weights is None else [float(np.float32(x)) for x in weights]
    n_boundary = 0
    for t in range(T):
        X = orol.stock_obs_batch(ocfg, st, mk)
        if t % mlp_every == 0:
            for mi, L_ in enumerate(L64):
                omlp.teacher_forced_layers(L_, X, g["mlp_hidden"][t, mi], g["mlp_out"][t, mi])
        for i in range(N):
            zs = [g["mlp_out"][t, mi, i].astype(np.float64) for mi in range(len(kinds))]
            sh, abar, ou[i] = orol.ensemble_shares_multi(kinds, zs, noise[t, :, i].astype(np.float64), ou[i],
                                                         weights=w)
            for k in range(K):
                if sh[k] != g["actions"][t, i, k]:
                    y = 100.0 * abar[k]
                    assert abs(abs(y - math.trunc(y)) - 0.5) < 1e-4, (t, i, k, y, g["actions"][t, i, k])
                    n_boundary += 1
        ostock.step(ocfg, st, mk, g["actions"][t])
        for i in range(N):
            if g["done"][t, i]:
                ou[i] = [[0.0] * K for _ in range(max(n_ddpg, 1))]
    return n_boundary


def test_weighted_ensemble_two_ddpg_members():
    """5 members (PPO, SAC, DDPG, DDPG, PPO) with Sharpe-softmax-like weights: two OU
    states (global-memory OU path), test windows advancing on reset."""
    fin = _fin()
    spec = [(1, fin.FIN_PPO_GAUSS, False), (2, fin.FIN_SAC_SQUASH, True), (3, fin.FIN_DDPG_OU, False),
            (5, fin.FIN_DDPG_OU, True), (6, fin.FIN_PPO_GAUSS, False)]
    w = np.array([0.35, 0.1, 0.25, 0.2, 0.1], dtype=np.float32)
    g, ocfg, mk, layers, kinds, noise = _run_stock(200, 12, spec, L=5, weights=w, window_offset=30,
                                                   advance_window_on_reset=True)
    _teacher_forced(g, ocfg, mk, layers, kinds, noise, weights=w)


def test_fifteen_member_ensemble():
    """Ensemble-2 of P:445 (5 PPO + 5 SAC + 5 DDPG), uniform mean; members 4.. take their
    biases and layer-1 shared term from L2; N = 300 (3 tiles, ragged)."""
    fin = _fin()
    spec = []
    for j in range(5):
        spec += [(10 + 3 * j, fin.FIN_PPO_GAUSS, j % 2 == 0), (11 + 3 * j, fin.FIN_SAC_SQUASH, j % 2 == 1),
                 (12 + 3 * j, fin.FIN_DDPG_OU, j == 4)]
    g, ocfg, mk, layers, kinds, noise = _run_stock(300, 7, spec, L=5, window_offset=30,
                                                   advance_window_on_reset=True)
    _teacher_forced(g, ocfg, mk, layers, kinds, noise, mlp_every=3)


def test_validate_and_weight_pipeline():
    """validate_and_weight: one deterministic validation rollout per member; the Sharpe
    ratios and weights must follow from the replayed validation equity (oracle metrics)
    and oracle.policy.softmax_weights."""
    import torch
    fin = _fin()
    from paper_2501_10709_b200 import ensemble
    rows, N, L, T = 150, 256, 5, 10
    m = market.stock_c1(rows=rows)
    kw = dict(num_envs=N, num_assets=30, num_indicators=8, num_rows=rows, episode_len=L, window_stride=5,
              window_offset=30, num_windows=(rows - 1 - L - 30) // 5 + 1, window_block=128,
              advance_window_on_reset=True)
    ocfg, fcfg = stock_pair(**kw)
    env = fin.fin_env_create(fcfg, m.market)
    kinds = [fin.FIN_PPO_GAUSS, fin.FIN_SAC_SQUASH, fin.FIN_DDPG_OU]
    layers = [spol.kaiming_bf16(spol.STOCK_DIMS, s) for s in (1, 2, 3)]
    pols = [fin.fin_policy_create(k, L_) for k, L_ in zip(kinds, layers)]
    w, sh, aggs = ensemble.validate_and_weight(env, pols, T, threshold=-0.5, temperature=0.7)
    w, sh, aggs = host(w), host(sh), host(aggs)
    # recompute: the same deterministic rollout per member logs its actions; the oracle
    # replays them and computes every episode's Sharpe
    sharpes = []
    for pol in pols:
        fin.fin_env_reset(env)
        a = zeros((T, N, 30), torch.int16)
        fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_NONE), fin.make_traj(actions=a))
        o, _ = ostock.run_actions(ocfg, m.market, host(a))
        tot, cnt = 0.0, 0
        for i in range(N):
            curves, _ = omet.split_episodes(1e6, o["asset"][:, i], o["done"][:, i])
            for cv in curves:
                s = omet.episode_metrics(cv)[1]
                if not math.isnan(s):
                    tot += s
                    cnt += 1
        sharpes.append(tot / cnt)
    np.testing.assert_allclose(sh, sharpes, rtol=1e-7)
    np.testing.assert_allclose(w, opol.softmax_weights(sharpes, -0.5, 0.7), rtol=1e-6, atol=1e-7)
    assert abs(w.sum() - 1.0) < 1e-6


# ------------------------------------------------------------------ crypto vote
@pytest.mark.parametrize("M", [3, 9])
def test_crypto_majority_vote(M):
    """DQN / Double DQN / Dueling DQN members (1:1:1), plurality vote with hold-preferring
    ties, epsilon-greedy with supplied uniforms.  M = 3: Q-nets resident in shared memory;
    M = 9 (Ensemble-2 of P:461): streamed."""
    import torch
    fin = _fin()
    T, N = 60 if M == 9 else 150, 300
    rows = market.crypto_market(T, seed=41)
    eps = float(np.float32(0.05))
    ocfg = ocry.CryptoEnvConfig(num_envs=N, episode_len=T)
    fcfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=T + 1,
                          episode_len=T, reward_scale=1.0, cost_rate=0.0, epsilon=eps)
    env = fin.fin_env_create(fcfg, rows)
    layers, kinds = [], []
    for j in range(M):
        kind = (fin.FIN_Q_ARGMAX, fin.FIN_Q_ARGMAX, fin.FIN_Q_DUELING)[j % 3]
        dims = spol.CRYPTO_DIMS if kind == fin.FIN_Q_ARGMAX else tuple(spol.CRYPTO_DIMS[:-1]) + (4,)
        layers.append(spol.random_bias(spol.kaiming_bf16(dims, 40 + j), 60 + j))
        kinds.append(kind)
    pols = [fin.fin_policy_create(k, L_) for k, L_ in zip(kinds, layers)]
    uni = inputs.crypto_uniforms(T, N, seed=44)
    logs = dict(actions=zeros((T, N, 1), torch.int16), hold=zeros((T, N, 1), torch.int16),
                cash=zeros((T, N), torch.float64), asset=zeros((T, N), torch.float64),
                reward=zeros((T, N), torch.float32), done=zeros((T, N), torch.uint8),
                mlp_out=zeros((T, M, N, 3), torch.float32), mlp_hidden=zeros((T, M, N, 2, 128), torch.int16))
    fin.fin_rollout(env, pols, T, fin.make_noise(fin.FIN_NOISE_SUPPLIED, 0, dev(uni)), fin.make_traj(**logs))
    g = {k: host(v) for k, v in logs.items()}
    assert fin.fin_env_check(env) == 0
    st = ocry.reset(ocfg)
    L64 = [omlp.layers_f64(L_) for L_ in layers]
    n_split = 0
    for t in range(T):
        X = orol.crypto_obs_batch(ocfg, st, rows)
        for mi, L_ in enumerate(L64):
            # (a dueling member logs its advantage head A_0..A_2, the first 3 of its 4 outputs)
            omlp.teacher_forced_layers(L_, X, g["mlp_hidden"][t, mi], g["mlp_out"][t, mi])
        for i in range(N):
            qs = [g["mlp_out"][t, mi, i].astype(np.float64) for mi in range(M)]
            a = orol.crypto_vote_action(qs, eps, float(uni[t, i, 0]), float(uni[t, i, 1]))
            assert a == g["actions"][t, i, 0], (t, i)
            votes = [opol.argmax_lowest(list(q)) for q in qs]
            n_split += len(set(votes)) > 1
        o = ocry.step(ocfg, st, rows, g["actions"][t, :, 0])
        assert np.array_equal(np.array(o["pos"]), g["hold"][t, :, 0])
        assert np.array_equal(np.array(o["cash"]), g["cash"][t])
    assert n_split > 0          # the members disagreed somewhere: the vote was exercised
