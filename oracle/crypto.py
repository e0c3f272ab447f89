"""Crypto trading environment oracle (test infrastructure only).

PAPER.md §3.1, §5.2.2 (discrete actions)
(epsilon 0.005), BASELINE.json configs[3] (single asset, actions {-1,0,1},
position limit +-1, max holding 120 steps, 10-level LOB) and the readings
R24-R28 of DESIGN.md:

  target = clamp(h + a, -1, +1); if h != 0 and tau >= max_hold: target = 0
  delta  = target - h;  buys walk the asks level by level (fill min(rem, size_l)
           at ask_l), any remainder past the displayed depth fills at the last
           level; sells walk the bids the same way; fee multiplies the notional
  tau'   = 0 if target == 0; tau + 1 if target == h != 0; 1 otherwise
  reward = (v' - v) * scale, v = b + h m_t, v' = b' + target m_{t+1}
  done   when the episode reaches its last row (one episode over the series)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MID, ASK_PX, ASK_SZ, BID_PX, BID_SZ, F0 = 0, 1, 11, 21, 31, 41
LEVELS = 10
FACTORS = 101


@dataclass
class CryptoEnvConfig:
    num_envs: int
    episode_len: int
    max_hold: int = 120
    pos_limit: int = 1
    initial_cash: float = 1e6
    cost_rate: float = 0.0
    reward_scale: float = 1.0
    autoreset: bool = True


@dataclass
class CryptoEnvState:
    cash: list
    pos: list
    tau: list
    t_ep: list


def reset(cfg: CryptoEnvConfig) -> CryptoEnvState:
    n = cfg.num_envs
    return CryptoEnvState([float(cfg.initial_cash)] * n, [0] * n, [0] * n, [0] * n)


def walk_book(row, px_off: int, sz_off: int, qty: float) -> float:
    """Notional of ``qty`` units walked through the 10 displayed levels (R25)."""
    rem = float(qty)
    notional = 0.0
    for lvl in range(LEVELS):
        size = float(row[sz_off + lvl])
        fill = rem if rem < size else size
        notional = notional + fill * float(row[px_off + lvl])
        rem = rem - fill
    if rem > 0.0:
        notional = notional + rem * float(row[px_off + LEVELS - 1])
    return notional


def step_one(cfg: CryptoEnvConfig, b: float, h: int, tau: int, row, row_next, a: int):
    """One crypto transition; returns (b', target, tau', v, v', r)."""
    target = max(-cfg.pos_limit, min(cfg.pos_limit, h + a))
    if h != 0 and tau >= cfg.max_hold:
        target = 0
    delta = target - h
    UP = 1.0 + cfg.cost_rate
    DN = 1.0 - cfg.cost_rate
    m = float(row[MID])
    v = b + h * m
    if delta > 0:
        b = b - walk_book(row, ASK_PX, ASK_SZ, delta) * UP
    elif delta < 0:
        b = b + walk_book(row, BID_PX, BID_SZ, -delta) * DN
    if target == 0:
        tau2 = 0
    elif target == h:
        tau2 = tau + 1
    else:
        tau2 = 1
    vn = b + target * float(row_next[MID])
    r = (vn - v) * cfg.reward_scale
    return b, target, tau2, v, vn, r


def observation(st: CryptoEnvState, rows: np.ndarray, i: int, max_hold: int = 120) -> list:
    """[h, tau / max_hold, f_1 .. f_101] (reading R24)."""
    t = st.t_ep[i]
    return [float(st.pos[i]), st.tau[i] / max_hold] + [float(x) for x in rows[t, F0:F0 + FACTORS]]


def step(cfg: CryptoEnvConfig, st: CryptoEnvState, rows: np.ndarray, actions):
    """Step all envs with actions in {-1, 0, 1}; returns per-env pre-reset outputs."""
    out = {k: [] for k in ("cash", "pos", "tau", "asset", "asset_prev", "reward", "done")}
    for i in range(cfg.num_envs):
        t = st.t_ep[i]
        b, tgt, tau2, v, vn, r = step_one(cfg, st.cash[i], st.pos[i], st.tau[i], rows[t], rows[t + 1],
                                          int(actions[i]))
        done = (t + 1) == cfg.episode_len
        for k, val in (("cash", b), ("pos", tgt), ("tau", tau2), ("asset", vn), ("asset_prev", v),
                       ("reward", r), ("done", done)):
            out[k].append(val)
        if done and cfg.autoreset:
            st.cash[i], st.pos[i], st.tau[i], st.t_ep[i] = float(cfg.initial_cash), 0, 0, 0
        else:
            st.cash[i], st.pos[i], st.tau[i], st.t_ep[i] = b, tgt, tau2, t + 1
    return out
