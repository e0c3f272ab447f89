"""Pins for the stock-env oracle (oracle/stock.py) -- CPU only.

Each test checks the oracle against something other than itself: hand-worked
steps (tests/golden), SPEC hand examples, closed forms / invariants named in
BASELINE.json north_star, exact rational brute force on tiny inputs.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import stock
from synth import inputs, market


def _cfg(K, cost, scale, **kw):
    return stock.StockEnvConfig(num_envs=1, num_assets=K, num_indicators=0, num_rows=2, episode_len=10,
                                cost_rate=cost, reward_scale=scale, **kw)


def test_worked_steps(golden):
    g = golden("stock_worked_steps.json")
    for c in g["cases"]:
        cfg = _cfg(len(c["h"]), c["cost"], c["scale"])
        b, h, v, vn, r, _, _ = stock.step_one(cfg, c["b"], c["h"], c["p"], c["p_next"], c["a"])
        e = c["expect"]
        if "b" in e:
            assert b == e["b"], c["name"]
        if "h" in e:
            assert h == e["h"], c["name"]
        if "v" in e:
            assert v == e["v"], c["name"]
        if "v_next" in e:
            assert vn == e["v_next"], c["name"]
        if "r" in e:
            assert r == e["r"], c["name"]
        if "r_approx" in e:
            assert r == pytest.approx(e["r_approx"], rel=1e-9), c["name"]


def test_fee_gap_is_cost_times_notional():
    """SPEC S:179 / S:203: 10 bps on notional 1000 lowers the reward by exactly 1.0."""
    z = _cfg(1, 0.0, 1.0)
    c = _cfg(1, 0.001, 1.0)
    r0 = stock.step_one(z, 1e6, [0], [100.0], [100.0], [10])[4]
    r1 = stock.step_one(c, 1e6, [0], [100.0], [100.0], [10])[4]
    assert r0 - r1 == 1.0
    # sell side: proceeds n p (1 - c): 5 shares at 40 -> fee 0.2
    r0 = stock.step_one(z, 0.0, [5], [40.0], [40.0], [-5])[4]
    r1 = stock.step_one(c, 0.0, [5], [40.0], [40.0], [-5])[4]
    assert r0 - r1 == pytest.approx(0.2, abs=1e-12)


def test_zero_cost_trade_conserves_wealth_at_trade_instant():
    """with zero cost, trading at p_t leaves v unchanged (reward = price P&L only)."""
    cfg = _cfg(3, 0.0, 1.0)
    rng = np.random.default_rng(0)
    for _ in range(200):
        p = [float(x) for x in rng.integers(1, 400, size=3) / 4.0]      # dyadic: exact
        b = float(rng.integers(0, 2000))
        h = [int(x) for x in rng.integers(0, 20, size=3)]
        a = [int(x) for x in rng.integers(-25, 26, size=3)]
        b2, h2, v, vn, r, _, _ = stock.step_one(cfg, b, h, p, p, a)
        assert vn == v


def test_exact_rational_brute_force_K1():
    """Every 3-step action sequence a in {-2..2}^3 for K=1 against Fraction arithmetic
    (no rounding at all) with dyadic prices, zero cost -- all float64 ops are exact."""
    cfg = _cfg(1, 0.0, 1.0)
    prices = [1.25, 0.75, 0.5, 1.0]
    for seq in itertools.product(range(-2, 3), repeat=3):
        b, h = 3.0, [1]
        fb, fh = Fraction(3), 1
        for t, a in enumerate(seq):
            p, pn = prices[t], prices[t + 1]
            b, h, v, vn, r, _, _ = stock.step_one(cfg, b, h, [p], [pn], [a])
            fp, fpn = Fraction(p), Fraction(pn)
            fv = fb + fh * fp
            if a < 0:
                n = min(-a, fh)
                fb += n * fp
                fh -= n
            elif a > 0:
                n = 0
                while n < a and (n + 1) * fp <= fb:
                    n += 1
                fb -= n * fp
                fh += n
            fvn = fb + fh * fpn
            assert Fraction(b) == fb and h[0] == fh and Fraction(r) == fvn - fv, (seq, t)


def test_brute_force_greedy_is_lexicographic_max():
    """K<=3, |a|<=4, dyadic prices, cash<=20, c=0: the buy phase equals the
    lexicographically largest feasible buy vector found by enumeration."""
    rng = np.random.default_rng(1)
    dy = [0.25, 0.5, 0.75, 1.25]
    for trial in range(300):
        K = int(rng.integers(1, 4))
        cfg = _cfg(K, 0.0, 1.0)
        p = [dy[int(i)] for i in rng.integers(0, 4, size=K)]
        b = float(rng.integers(0, 21)) / 4.0
        h = [int(x) for x in rng.integers(0, 4, size=K)]
        a = [int(x) for x in rng.integers(-4, 5, size=K)]
        b2, h2, *_ = stock.step_one(cfg, b, h, p, p, a)
        # exact: sells first
        cash = Fraction(b)
        hh = list(h)
        for k in range(K):
            if a[k] < 0:
                n = min(-a[k], hh[k])
                cash += n * Fraction(p[k])
                hh[k] -= n
        ranges = [range(0, max(a[k], 0) + 1) for k in range(K)]
        feas = [v for v in itertools.product(*ranges)
                if sum(v[k] * Fraction(p[k]) for k in range(K)) <= cash]
        best = max(feas)  # tuple order is lexicographic
        assert [h2[k] - hh[k] for k in range(K)] == list(best), (trial, p, b, h, a)


def test_affordable_is_largest_count():
    rng = np.random.default_rng(2)
    for _ in range(2000):
        u = float(rng.uniform(1, 500)) * 1.001
        b = float(rng.uniform(0, 5000))
        want = int(rng.integers(0, 100))
        n = stock.affordable(b, u, want)
        assert 0 <= n <= want
        assert n * u <= b
        if n < want:
            assert (n + 1) * u > b


def _c0_env(N=8, **kw):
    m = market.stock_c0()
    cfg = stock.StockEnvConfig(num_envs=N, num_assets=4, num_indicators=4, num_rows=m.rows, episode_len=64, **kw)
    return cfg, m.market


def test_c0_invariants():
    """north_star invariants on C0: v = b + sum h p at every step; b >= 0, h >= 0;
    telescoping sum of rewards; exactly one done per episode."""
    cfg, mk = _c0_env()
    acts = inputs.stock_actions(64, 8, 4, seed=12)
    out, _ = stock.run_actions(cfg, mk, acts)
    for t in range(64):
        pn = mk[t + 1, 0, :].astype(np.float64)
        p = mk[t, 0, :].astype(np.float64)
        for i in range(8):
            b, h = out["cash"][t, i], out["hold"][t, i]
            assert b >= 0 and np.all(h >= 0)
            exact = math.fsum([b] + [float(h[k]) * float(pn[k]) for k in range(4)])
            assert out["asset"][t, i] == pytest.approx(exact, rel=1e-14)
            if t > 0:
                assert out["asset_prev"][t, i] == out["asset"][t - 1, i]   # v_t = v'_{t-1} bitwise
            # the executed change equals the supplied action where not clipped
            ex = out["executed"][t, i]
            assert np.all(np.abs(ex) <= 100)
    # telescoping: sum_t (v'_t - v_t) = v'_L - v_0 ; each subtraction is exact (Sterbenz)
    for i in range(8):
        s = math.fsum(out["reward"][:, i]) * 4096.0
        assert s == pytest.approx(out["asset"][-1, i] - 1e6, abs=1e-6)
    assert out["done"].sum(axis=0).tolist() == [1] * 8 and out["done"][-1].all()


def test_zero_actions_leave_assets_unchanged():
    cfg, mk = _c0_env()
    out, _ = stock.run_actions(cfg, mk, np.zeros((64, 8, 4), dtype=np.int16))
    assert np.all(out["cash"] == 1e6) and np.all(out["asset"] == 1e6) and np.all(out["reward"] == 0.0)


def test_batch_and_partition_independence():
    """S:216 / S:741: each env of a batch equals the env run alone (global ids via env_offset)."""
    m = market.stock_c1(rows=80)
    kw = dict(num_assets=30, num_indicators=8, num_rows=80, episode_len=5, window_stride=5,
              num_windows=10, window_block=2, advance_window_on_reset=True)
    acts = inputs.stock_actions(12, 6, 30, seed=5)
    full, _ = stock.run_actions(stock.StockEnvConfig(num_envs=6, **kw), m.market, acts)
    for lo, hi in ((0, 3), (3, 6), (4, 5)):
        part, _ = stock.run_actions(stock.StockEnvConfig(num_envs=hi - lo, env_offset=lo, **kw),
                                    m.market, acts[:, lo:hi])
        for key in ("cash", "hold", "asset", "reward", "done"):
            assert np.array_equal(part[key], full[key][:, lo:hi]), key


def test_clamp_and_flag_out_of_range():
    cfg = _cfg(2, 0.0, 1.0)
    b, h, v, vn, r, aa, oor = stock.step_one(cfg, 1e9, [0, 500], [1.0, 1.0], [1.0, 1.0], [300, -250])
    assert aa == [100, -100] and oor and h == [100, 400]


def test_hold_cap_int16():
    cfg = _cfg(1, 0.0, 1.0)
    b, h, *_ = stock.step_one(cfg, 1e9, [32700], [1.0], [1.0], [100])
    assert h == [stock.HOLD_MAX]


def test_autoreset_and_window_advance():
    m = market.stock_c1(rows=60)
    cfg = stock.StockEnvConfig(num_envs=3, num_assets=30, num_indicators=8, num_rows=60, episode_len=5,
                               window_stride=5, window_offset=30, num_windows=3, window_block=1,
                               advance_window_on_reset=True)
    st = stock.reset(cfg)
    assert st.window == [0, 1, 2]
    acts = inputs.stock_actions(10, 3, 30, seed=3)
    out, st = stock.run_actions(cfg, m.market, acts, st)
    assert out["done"][4].all() and out["done"][9].all() and out["done"].sum() == 6
    assert st.window == [2, 0, 1]
    assert st.t_ep == [0, 0, 0] and st.cash == [1e6] * 3


def test_no_autoreset_raises_episode_finished():
    cfg, mk = _c0_env(N=1, autoreset=False)
    cfg.episode_len = 2
    st = stock.reset(cfg)
    z = np.zeros((1, 4), dtype=np.int16)
    stock.step(cfg, st, mk, z)
    o = stock.step(cfg, st, mk, z)
    assert o["done"] == [True]
    with pytest.raises(RuntimeError):
        stock.step(cfg, st, mk, z)
