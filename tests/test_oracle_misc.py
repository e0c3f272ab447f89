"""Pins for oracle/metrics.py, oracle/crypto.py, oracle/philox.py and synth/ -- CPU only."""
import math

import numpy as np
import pytest

from oracle import crypto, metrics, philox
from synth import market


# ------------------------------------------------------------------ metrics
def test_metric_examples(golden):
    for c in golden("metrics_examples.json")["cases"]:
        eq = c["equity"]
        assert metrics.cumulative_return(eq) == pytest.approx(c["cum"], abs=1e-15)
        assert metrics.max_drawdown(eq) == pytest.approx(c["mdd"], abs=1e-15)
        if "drawdown" in c:
            assert metrics.drawdown_curve(eq) == c["drawdown"]
        if "sharpe" in c:
            s = metrics.sharpe(eq)
            if c["sharpe"] == "nan":
                assert math.isnan(s)
            else:
                assert s == pytest.approx(c["sharpe"], abs=c["sharpe_tol"])


def test_mdd_brute_force_and_monotone():
    rng = np.random.default_rng(0)
    for _ in range(200):
        eq = list(np.exp(np.cumsum(rng.normal(0, 0.05, int(rng.integers(1, 40))))))
        brute = min([eq[j] / eq[i] - 1.0 for i in range(len(eq)) for j in range(i, len(eq))])
        assert metrics.max_drawdown(eq) == pytest.approx(brute, abs=1e-15)
        assert metrics.max_drawdown(eq) <= 0.0
    assert metrics.drawdown_curve([1.0, 2.0, 3.0]) == [0.0, 0.0, 0.0]


def test_sharpe_against_library_and_short_episode():
    rng = np.random.default_rng(1)
    eq = list(1e6 * np.exp(np.cumsum(rng.normal(0, 0.01, 31))))
    r = np.array(eq[1:]) / np.array(eq[:-1]) - 1
    assert metrics.sharpe(eq) == pytest.approx(math.sqrt(252) * r.mean() / r.std(ddof=1), rel=1e-12)
    assert math.isnan(metrics.sharpe([1.0, 2.0]))           # one return: std undefined
    assert metrics.cumulative_return([4.0, 1.0, 5.0]) == 0.25


def test_split_episodes():
    done, rest = metrics.split_episodes(10.0, [11.0, 12.0, 9.0, 10.5], [False, True, False, False])
    assert done == [[10.0, 11.0, 12.0]] and rest == [10.0, 9.0, 10.5]


# ------------------------------------------------------------------ crypto
def _row(mid=100.0, asks=(101.0, 102.0, 103.0), asz=(0.4, 0.3, 0.5), bids=(99.0, 98.0, 97.0), bsz=(0.4, 0.3, 0.5)):
    r = np.zeros(144, dtype=np.float64)
    r[crypto.MID] = mid
    for i in range(10):
        r[crypto.ASK_PX + i] = asks[min(i, len(asks) - 1)] + max(0, i - len(asks) + 1)
        r[crypto.BID_PX + i] = bids[min(i, len(bids) - 1)] - max(0, i - len(bids) + 1)
        r[crypto.ASK_SZ + i] = asz[i] if i < len(asz) else 0.0
        r[crypto.BID_SZ + i] = bsz[i] if i < len(bsz) else 0.0
    return r


def test_book_walk_hand_example():
    """1 unit through sizes (0.4, 0.3, 0.5) at (p1, p2, p3) costs 0.4 p1 + 0.3 p2 + 0.3 p3."""
    r = _row()
    assert crypto.walk_book(r, crypto.ASK_PX, crypto.ASK_SZ, 1) == pytest.approx(0.4 * 101 + 0.3 * 102 + 0.3 * 103, rel=1e-15)
    assert crypto.walk_book(r, crypto.BID_PX, crypto.BID_SZ, 1) == pytest.approx(0.4 * 99 + 0.3 * 98 + 0.3 * 97, rel=1e-15)
    # beyond the displayed depth (1.2 units shown) the remainder fills at the last level
    last = r[crypto.ASK_PX + 9]
    assert crypto.walk_book(r, crypto.ASK_PX, crypto.ASK_SZ, 2) == pytest.approx(
        0.4 * 101 + 0.3 * 102 + 0.5 * 103 + 0.8 * last, rel=1e-15)


def test_crypto_position_rules():
    cfg = crypto.CryptoEnvConfig(num_envs=1, episode_len=1000)
    r = _row()
    # flat with zero action: v constant, reward 0
    b, tgt, tau, v, vn, rew = crypto.step_one(cfg, 1e6, 0, 0, r, r, 0)
    assert (b, tgt, tau, rew) == (1e6, 0, 0, 0.0)
    # position limit: long + buy stays long
    b, tgt, tau, *_ = crypto.step_one(cfg, 1e6, 1, 5, r, r, 1)
    assert tgt == 1 and tau == 6 and b == 1e6
    # flip from short to long: delta = 2, tau restarts at 1
    b, tgt, tau, *_ = crypto.step_one(cfg, 1e6, -1, 7, r, r, 1)
    assert tgt == 0 and tau == 0
    # forced exit at max_hold overrides the action
    b, tgt, tau, *_ = crypto.step_one(cfg, 1e6, 1, 120, r, r, 1)
    assert tgt == 0 and tau == 0
    b, tgt, tau, *_ = crypto.step_one(cfg, 1e6, 1, 119, r, r, 0)
    assert tgt == 1 and tau == 120


def test_crypto_invariants_random_walk():
    rows = market.crypto_market(400, seed=3)
    cfg = crypto.CryptoEnvConfig(num_envs=16, episode_len=400)
    st = crypto.reset(cfg)
    rng = np.random.default_rng(2)
    for t in range(400):
        o = crypto.step(cfg, st, rows, rng.integers(-1, 2, 16))
        assert all(abs(p) <= 1 for p in o["pos"]) and all(0 <= x <= 120 for x in o["tau"])
        for i in range(16):
            assert o["asset"][i] == pytest.approx(o["cash"][i] + o["pos"][i] * float(rows[t + 1, 0]), rel=1e-15)
            assert o["cash"][i] > 0
    assert all(o["done"])


# ------------------------------------------------------------------ philox
def test_philox_known_answers(golden):
    for c in golden("philox_kat.json")["cases"]:
        ctr = [int(x, 16) for x in c["ctr"]]
        key = [int(x, 16) for x in c["key"]]
        assert list(philox.philox4x32_10(ctr, key)) == [int(x, 16) for x in c["out"]]


def test_philox_normals_statistics():
    z = []
    for g in range(3000):
        z.extend(philox.stock_noise(1234, g, 7, 0, 8))
    z = np.array(z)
    n = len(z)
    assert abs(z.mean()) < 4 / math.sqrt(n) and abs(z.var() - 1) < 4 * math.sqrt(2 / n)
    # KS against N(0,1)
    from scipy import stats
    assert stats.kstest(z, "norm").pvalue > 1e-3


# ------------------------------------------------------------------ synthetic inputs
def test_gbm_closed_form_sigma0_and_determinism():
    rng = np.random.default_rng(0)
    s0 = np.array([100.0, 60.0])
    path = market.gbm_close(50, 2, rng, mu=2e-4, sigma=0.0, s0=s0)
    d = np.arange(51)[:, None]
    np.testing.assert_allclose(path, s0 * np.exp(2e-4 * d), rtol=1e-12)
    a, b = market.stock_c0(), market.stock_c0()
    assert a.market.tobytes() == b.market.tobytes()
    assert market.stock_c0(seed=12).market.tobytes() != a.market.tobytes()


def test_indicator_special_cases():
    x = np.array([[1.0], [2.0], [3.0], [4.0]])
    assert market.sma(x, 3)[2:, 0].tolist() == [2.0, 3.0]
    assert np.all(market.rsi(np.arange(1.0, 60.0)[:, None])[1:] == 100.0)
    assert np.all(np.abs(market.macd(np.full((40, 1), 7.0))) < 1e-12)
    const = np.full((40, 1), 5.0)
    assert np.all(market.cci(const, const, const) == 0.0)


def test_bar_invariants_and_shapes():
    m = market.stock_c1(rows=100)
    o, h, l_, c = m.open_all, m.high_all, m.low_all, m.close_all
    assert np.all(l_ <= np.minimum(o, c)) and np.all(np.maximum(o, c) <= h)
    assert m.market.shape == (100, 10, 30) and m.market.dtype == np.float32
    assert 1 + 30 + 30 + 30 * 8 == 301
    assert np.all(m.market[0, 1] == 1.0)
    z = m.market[:, 2:, :].astype(np.float64)
    assert np.all(np.abs(z.mean(axis=0)) < 1e-5)


def test_crypto_market_shape_and_book_order():
    rows = market.crypto_market(1000, seed=41)
    assert rows.shape == (1001, 144) and rows.dtype == np.float32
    ask = rows[:, 1:11]
    bid = rows[:, 21:31]
    assert np.all(np.diff(ask, axis=1) >= 0) and np.all(np.diff(bid, axis=1) <= 0)
    assert np.all(bid[:, 0] < rows[:, 0]) and np.all(rows[:, 0] < ask[:, 0])
    f = rows[:, 41:142].astype(np.float64)
    assert abs(f.std() - 1.0) < 0.15
    lag = np.mean([np.corrcoef(f[:-1, j], f[1:, j])[0, 1] for j in range(101)])
    assert abs(lag - 0.9) < 0.05
