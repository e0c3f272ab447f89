"""Stock trading environment oracle (test infrastructure only).

Follows PAPER.md §3.1 and §4.2:
  state  s_t = [b_t, p_t, h_t, f_t]
  action a_t = change in position, h_{t+1} = h_t + a_t
  reward R = v_{t+1} - v_t,  v_t = b_t + p_t^T h_t
  reset  s_t -> s_0 ; step (s_t, a_t) -> s_{t+1}; reward (s_t, a_t, s_{t+1}) -> r_t
with transaction costs ("0.1% per side", BASELINE.json configs[0]) and the
readings of DESIGN.md §3 (R2 execute at p_t / mark at p_{t+1}; R3 sells first, then
buys in ascending asset order; R4 fees; R5 affordability; R6 clamp; R8 reward
scale 2^-12; R9 episode length; R10 windows; R-HOLD int16 holdings cap).

Every arithmetic step is one IEEE binary64 operation on Python floats, in the
order written (CPython never fuses a*b+c).  Explicit loops over env and asset.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

HOLD_MAX = 32767  # holdings are stored as int16 (reading R-HOLD)


@dataclass
class StockEnvConfig:
    num_envs: int
    num_assets: int
    num_indicators: int
    num_rows: int
    episode_len: int                 # L_ep steps per episode (R9)
    window_stride: int = 5           # R10: window w starts at window_offset + w*window_stride
    window_offset: int = 0
    num_windows: int = 1
    window_block: int = 128          # envs g in [j*block, (j+1)*block) share a window
    window_base: int = 0
    advance_window_on_reset: bool = False   # C2 test mode: w <- (w+1) mod W on reset
    max_trade: int = 100
    initial_cash: float = 1e6
    cost_rate: float = 1e-3
    reward_scale: float = 2.0 ** -12
    autoreset: bool = True
    env_offset: int = 0              # global id of local env 0 (partitioning)


@dataclass
class StockEnvState:
    cash: list                       # b per env (float)
    hold: list                       # h[env][k] (int)
    t_ep: list                       # step within episode
    window: list                     # window index per env
    done_flag: list = field(default_factory=list)   # only meaningful with autoreset=False


def window_of(cfg: StockEnvConfig, g: int) -> int:
    """R10: w_g = (w_base + floor(g / window_block)) mod W."""
    return (cfg.window_base + g // cfg.window_block) % cfg.num_windows


def window_start(cfg: StockEnvConfig, w: int) -> int:
    return cfg.window_offset + w * cfg.window_stride


def reset(cfg: StockEnvConfig) -> StockEnvState:
    """P:211 reset: b = initial cash, h = 0, t_ep = 0."""
    n = cfg.num_envs
    return StockEnvState(cash=[float(cfg.initial_cash)] * n,
                         hold=[[0] * cfg.num_assets for _ in range(n)],
                         t_ep=[0] * n,
                         window=[window_of(cfg, cfg.env_offset + i) for i in range(n)],
                         done_flag=[False] * n)


def total_asset(b: float, h, p) -> float:
    """v = b + p^T h, accumulated in ascending asset order."""
    v = b
    for k in range(len(h)):
        v = v + h[k] * p[k]
    return v


def affordable(b: float, u: float, want: int) -> int:
    """R5: the largest n in [0, want] with fl(n*u) <= b.

    fl(n*u) is non-decreasing in n (rounding is monotone), so the predicate is
    monotone and a binary search finds the largest n that satisfies it.
    """
    if want <= 0:
        return 0
    lo, hi = 0, want           # invariant: fl(lo*u) <= b (lo = 0 always affordable when b >= 0)
    if not (0.0 <= b):
        return 0
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if mid * u <= b:
            lo = mid
        else:
            hi = mid - 1
    return lo


def step_one(cfg: StockEnvConfig, b: float, h: list, p: list, p_next: list, a: list):
    """One transition of one env (SURVEY §8(c) c.3 with reading R5).

    Returns (b', h', v, v', r, a_clamped, out_of_range) -- all pre-reset.
    """
    c = cfg.cost_rate
    UP = 1.0 + c
    DN = 1.0 - c
    K = cfg.num_assets
    h = list(h)
    # 1. total asset at the state's price
    v = total_asset(b, h, p)
    # 2. clamp the action to +-max_trade (R6)
    aa = []
    oor = False
    for k in range(K):
        ak = int(a[k])
        if ak > cfg.max_trade:
            ak, oor = cfg.max_trade, True
        if ak < -cfg.max_trade:
            ak, oor = -cfg.max_trade, True
        aa.append(ak)
    # 3. sells, clipped to holdings, proceeds n p (1 - c)   (R3, R4)
    for k in range(K):
        if aa[k] < 0:
            n = min(-aa[k], h[k])
            b = b + (n * p[k]) * DN
            h[k] = h[k] - n
    # 4. buys in ascending asset order at u = p (1 + c), clipped to what the cash affords (R3-R5)
    for k in range(K):
        if aa[k] > 0:
            u = p[k] * UP
            n = affordable(b, u, min(aa[k], HOLD_MAX - h[k]))
            b = b - n * u
            h[k] = h[k] + n
    # 5. mark at the next row's price (R2)
    v_next = total_asset(b, h, p_next)
    # 6. reward = (v' - v) * 2^-12 (R8)
    r = (v_next - v) * cfg.reward_scale
    return b, h, v, v_next, r, aa, oor


def market_close(market: np.ndarray, d: int):
    return [float(x) for x in market[d, 0, :]]


def step(cfg: StockEnvConfig, st: StockEnvState, market: np.ndarray, actions: np.ndarray):
    """VecEnv step over all envs.  ``actions`` int [N][K].

    Returns a dict of per-env outputs of this transition (pre-reset values):
    cash, hold, asset (v'), asset_prev (v), reward, done, executed (h' - h).
    The state is advanced in place; with autoreset a done env is reset (and in
    test mode its window advances) so the next step starts from s_0.
    """
    N = cfg.num_envs
    out = {k: [] for k in ("cash", "hold", "asset", "asset_prev", "reward", "done", "executed", "oor")}
    for i in range(N):
        if not cfg.autoreset and st.done_flag[i]:
            raise RuntimeError("EpisodeFinished: stepping a done env without autoreset (S:165)")
        d = window_start(cfg, st.window[i]) + st.t_ep[i]
        p = market_close(market, d)
        pn = market_close(market, d + 1)
        h0 = st.hold[i]
        b, h, v, vn, r, aa, oor = step_one(cfg, st.cash[i], h0, p, pn, list(actions[i]))
        t = st.t_ep[i] + 1
        done = t == cfg.episode_len
        out["cash"].append(b)
        out["hold"].append(list(h))
        out["asset"].append(vn)
        out["asset_prev"].append(v)
        out["reward"].append(r)
        out["done"].append(done)
        out["executed"].append([h[k] - h0[k] for k in range(cfg.num_assets)])
        out["oor"].append(oor)
        if done and cfg.autoreset:
            st.cash[i] = float(cfg.initial_cash)
            st.hold[i] = [0] * cfg.num_assets
            st.t_ep[i] = 0
            if cfg.advance_window_on_reset:
                st.window[i] = (st.window[i] + 1) % cfg.num_windows
        else:
            st.cash[i] = b
            st.hold[i] = h
            st.t_ep[i] = t
            st.done_flag[i] = done
    return out


def observation(cfg: StockEnvConfig, st: StockEnvState, market: np.ndarray, i: int) -> list:
    """Unquantised float64 observation of env i (reading R13/R14):
    x = [b / b0, close_norm[d][k] (k<K), h_k / max_trade (k<K), feat[d][j][k] in
    indicator-major order j*K + k]."""
    d = window_start(cfg, st.window[i]) + st.t_ep[i]
    K, I = cfg.num_assets, cfg.num_indicators
    x = [st.cash[i] / cfg.initial_cash]
    x += [float(market[d, 1, k]) for k in range(K)]
    x += [st.hold[i][k] / cfg.max_trade for k in range(K)]
    for j in range(I):
        x += [float(market[d, 2 + j, k]) for k in range(K)]
    return x


def run_actions(cfg: StockEnvConfig, market: np.ndarray, actions: np.ndarray, st: StockEnvState | None = None):
    """Replay supplied int actions [T][N][K] from reset (or ``st``); stack the outputs [T][N]..."""
    if st is None:
        st = reset(cfg)
    T = actions.shape[0]
    res = {k: [] for k in ("cash", "hold", "asset", "asset_prev", "reward", "done", "executed", "oor")}
    for t in range(T):
        o = step(cfg, st, market, actions[t])
        for k in res:
            res[k].append(o[k])
    arr = {
        "cash": np.array(res["cash"], dtype=np.float64),
        "hold": np.array(res["hold"], dtype=np.int64),
        "asset": np.array(res["asset"], dtype=np.float64),
        "asset_prev": np.array(res["asset_prev"], dtype=np.float64),
        "reward": np.array(res["reward"], dtype=np.float64),
        "done": np.array(res["done"], dtype=bool),
        "executed": np.array(res["executed"], dtype=np.int64),
        "oor": np.array(res["oor"], dtype=bool),
    }
    return arr, st


def is_finite_market(market: np.ndarray) -> bool:
    return bool(np.all(np.isfinite(market))) and bool(np.all(market[:, 0, :] > 0))


__all__ = ["StockEnvConfig", "StockEnvState", "reset", "step", "step_one", "run_actions",
           "observation", "total_asset", "affordable", "window_of", "window_start", "HOLD_MAX",
           "math"]
