"""Rollout drivers for the oracle (test infrastructure only).

The producer side of PAPER.md §3.2 / Fig. P:164-171 and §4.3 (T x N x D sample
tensors): for t < T, a_t ~ pi(s_t) (policy forward + sampling), then
VecEnv step/reward/reset.  Each function composes the per-step oracles of
``stock`` / ``crypto`` / ``mlp`` / ``policy`` in that order.
"""
from __future__ import annotations

import numpy as np

from . import crypto as cry
from . import mlp, policy, stock

# member kinds (mirrors the names used in DESIGN.md, not any GPU header)
PPO_GAUSS, SAC_SQUASH, DDPG_OU, Q_ARGMAX = 0, 1, 2, 3


def stock_obs_batch(cfg: stock.StockEnvConfig, st: stock.StockEnvState, market) -> np.ndarray:
    return np.array([stock.observation(cfg, st, market, i) for i in range(cfg.num_envs)], dtype=np.float64)


def member_action(kind: int, z: float, eps: float, ou_x: float):
    """Continuous action of one member for one asset; returns (a, new_ou_x)."""
    if kind == PPO_GAUSS:
        return policy.gaussian_action(z, eps), ou_x
    if kind == SAC_SQUASH:
        return policy.sac_action(z, eps), ou_x
    if kind == DDPG_OU:
        x = policy.ou_update(ou_x, eps)
        return policy.ddpg_action(z, x), x
    raise ValueError(kind)


def ensemble_shares_multi(kinds, zs, eps, ou_slots, max_trade: int = 100, weights=None):
    """zs[m][K], eps[m][K], ou_slots[j][K] (state of the j-th DDPG member, in member
    order) -> (shares[K], abar[K], ou_slots').  Executed action: the uniform mean of the
    members' continuous actions (reading R20), or the weights' weighted sum (the
    Sharpe-softmax weights of PAPER.md P:309, reading R-GATE)."""
    K = len(zs[0])
    ou_slots = [list(x) for x in ou_slots]
    out, abar = [], []
    for k in range(K):
        acts = []
        j = 0
        for m, kind in enumerate(kinds):
            x_old = ou_slots[j][k] if kind == DDPG_OU else 0.0
            a, x = member_action(kind, float(zs[m][k]), float(eps[m][k]), x_old)
            if kind == DDPG_OU:
                ou_slots[j][k] = x
                j += 1
            acts.append(a)
        mean = policy.ensemble_mean(acts) if weights is None else policy.weighted_mean(acts, weights)
        abar.append(mean)
        out.append(policy.shares(mean, max_trade))
    return out, abar, ou_slots


def ensemble_shares(kinds, zs, eps, ou, max_trade: int = 100, weights=None):
    """zs[m][K], eps[m][K], ou[K] (the single DDPG member's state) -> (shares[K], abar[K], ou')."""
    out, abar, slots = ensemble_shares_multi(kinds, zs, eps, [list(ou)], max_trade, weights)
    return out, abar, slots[0]


def crypto_vote_action(qs, epsilon: float = 0.0, u_explore: float = 1.0, u_action: float = 0.0) -> int:
    """Crypto ensemble: each member's greedy action (argmax of its
    first 3 outputs -- Q for DQN / Double DQN, the advantage head for Dueling DQN) is a
    vote; the plurality winner (ties to hold, then the lowest index) is then subject to
    epsilon-greedy exploration like a single agent.  Returns the action in {-1, 0, 1}."""
    votes = [policy.argmax_lowest(list(q[:3])) - 1 for q in qs]
    a = policy.majority_vote(votes)
    if u_explore < epsilon:
        return min(int(u_action * 3), 2) - 1
    return a


def stock_policy_rollout(cfg: stock.StockEnvConfig, market, members, kinds, noise, T: int,
                         st: stock.StockEnvState | None = None, weights=None):
    """Free-running float64 rollout: members = [layers], noise [T][M][N][K] (supplied mode).

    Returns dict of [T][N](...) arrays: actions, z [T][M][N][K], reward, done, cash, hold, asset.
    """
    if st is None:
        st = stock.reset(cfg)
    N, K, M = cfg.num_envs, cfg.num_assets, len(members)
    L64 = [mlp.layers_f64(m) for m in members]
    ou = [[0.0] * K for _ in range(N)]
    log = {k: [] for k in ("actions", "z", "reward", "done", "cash", "hold", "asset")}
    for t in range(T):
        X = stock_obs_batch(cfg, st, market)
        zs = [mlp.forward(L, X) for L in L64]   # [M][N][K]
        acts = []
        for i in range(N):
            sh, _, ou[i] = ensemble_shares(kinds, [zs[m][i] for m in range(M)],
                                           [noise[t][m][i] for m in range(M)], ou[i], cfg.max_trade, weights)
            acts.append(sh)
        acts = np.array(acts, dtype=np.int64)
        o = stock.step(cfg, st, market, acts)
        for i in range(N):
            if o["done"][i] and cfg.autoreset:
                ou[i] = [0.0] * K
        log["actions"].append(acts)
        log["z"].append(np.stack(zs))
        log["reward"].append(o["reward"])
        log["done"].append(o["done"])
        log["cash"].append(o["cash"])
        log["hold"].append(o["hold"])
        log["asset"].append(o["asset"])
    return {k: np.array(v) for k, v in log.items()}, st


def crypto_obs_batch(cfg: cry.CryptoEnvConfig, st: cry.CryptoEnvState, rows) -> np.ndarray:
    return np.array([cry.observation(st, rows, i, cfg.max_hold) for i in range(cfg.num_envs)], dtype=np.float64)


def crypto_q_rollout(cfg: cry.CryptoEnvConfig, rows, layers, T: int, epsilon: float = 0.0,
                     uniforms=None, st: cry.CryptoEnvState | None = None):
    """Free-running Q-argmax rollout (epsilon-greedy with supplied uniforms [T][N][2])."""
    if st is None:
        st = cry.reset(cfg)
    L64 = mlp.layers_f64(layers)
    log = {k: [] for k in ("actions", "q", "reward", "done", "cash", "pos", "tau", "asset")}
    for t in range(T):
        X = crypto_obs_batch(cfg, st, rows)
        q = mlp.forward(L64, X)
        acts = []
        for i in range(cfg.num_envs):
            if uniforms is not None:
                j = policy.epsilon_greedy(list(q[i]), epsilon, float(uniforms[t][i][0]), float(uniforms[t][i][1]))
            else:
                j = policy.argmax_lowest(list(q[i]))
            acts.append(j - 1)
        o = cry.step(cfg, st, rows, acts)
        log["actions"].append(acts)
        log["q"].append(q)
        for k in ("reward", "done", "cash", "pos", "tau", "asset"):
            log[k].append(o[k])
    return {k: np.array(v) for k, v in log.items()}, st
