"""Pins for oracle/market.py (market preparation) -- CPU only.

SPEC S:65-67 examples, closed forms and special cases of each indicator, the
perturbation properties of SPEC S:70-78 (identity at 0, returns unchanged, seeded
determinism), scale invariance of the z-scored features, and a cross-check against the
independent numpy fixture generator of synth/market.py.
"""
import math

import numpy as np
import pytest

from oracle import market as om
from synth import market as sm


def test_spec_examples():
    assert om.sma([1.0, 2.0, 3.0, 4.0], 3)[2:] == [2.0, 3.0]
    assert all(v == 100.0 for v in om.rsi([float(x) for x in range(1, 50)], 14)[1:])
    assert om.macd([7.5] * 40) == [0.0] * 40


def test_indicator_closed_forms():
    c = [100.0 + d for d in range(80)]
    assert om.sma(c, 30)[-1] == pytest.approx(sum(c[-30:]) / 30, abs=1e-12)
    # EMA of a geometric sequence started at x0: e_d = x0 (1-a)^d + a sum ... -> closed form check on a step
    e = om.ema([0.0] + [1.0] * 50, 0.25)
    assert e[-1] == pytest.approx(1.0 - 0.75 ** 50, abs=1e-15)
    # Bollinger of a constant series collapses on the SMA; CCI and DX of a constant series are 0
    assert om.bollinger([3.0] * 30, True) == [3.0] * 30 and om.bollinger([3.0] * 30, False) == [3.0] * 30
    assert om.cci([2.0] * 40, [1.0] * 40, [1.5] * 40) == [0.0] * 40
    assert om.dx([2.0] * 40, [1.0] * 40, [1.5] * 40) == [0.0] * 40
    # RSI of a strictly decreasing series is 0 after day 0; population std of [1, 3] is 1
    assert all(v == 0.0 for v in om.rsi([float(50 - x) for x in range(40)], 30)[1:])
    assert om._window_pstd([1.0, 3.0], 1, 20) == 1.0
    # DX of a pure up-trend (highs and lows rising by 1, closes inside) is 100
    h = [10.0 + d for d in range(40)]
    l_ = [9.0 + d for d in range(40)]
    assert all(v == pytest.approx(100.0) for v in om.dx(h, l_, [9.5 + d for d in range(40)])[1:])
    z = om.zscore([1.0, 2.0, 3.0])
    assert z == pytest.approx([-math.sqrt(1.5), 0.0, math.sqrt(1.5)], abs=1e-15)
    assert om.zscore([4.0, 4.0]) == [0.0, 0.0]


def _ohlcv(K=5, rows=80, seed=3):
    m = sm.stock_market(K=K, rows=rows, seed=seed)
    x = np.stack([m.open_all, m.high_all, m.low_all, m.close_all[1:] if m.close_all.shape[0] > m.open_all.shape[0]
                  else m.close_all, m.volume_all], axis=1).astype(np.float32)
    return m, x


def test_matches_independent_fixture_generator():
    """synth/market.py builds the same tensor with numpy (different code, same
    definitions): raw indicators agree to 1e-9 relative, the f32 tensor to a few ulp."""
    m, x = _ohlcv()
    x64 = np.stack([m.open_all, m.high_all, m.low_all, m.close_all, m.volume_all], axis=1)
    mk, raw = om.prepare_stock_market(x64, sm.WARMUP_DAYS)
    np.testing.assert_allclose(raw, m.raw_indicators, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(mk, m.market, rtol=2e-6, atol=2e-6)


def test_perturbation_properties():
    m, x = _ohlcv(K=4, rows=60)
    base, raw0 = om.prepare_stock_market(x, sm.WARMUP_DAYS, magnitude=0.0, seed=9)
    same, _ = om.prepare_stock_market(x, sm.WARMUP_DAYS, magnitude=0.0, seed=123)
    assert np.array_equal(base, same)                                   # magnitude 0: identity
    p1, raw1 = om.prepare_stock_market(x, sm.WARMUP_DAYS, magnitude=0.01, seed=9)
    p2, _ = om.prepare_stock_market(x, sm.WARMUP_DAYS, magnitude=0.01, seed=9)
    assert np.array_equal(p1, p2)                                       # seeded determinism
    c0 = base[:, 0, :].astype(np.float64)
    c1 = p1[:, 0, :].astype(np.float64)
    f = c1 / c0
    assert np.all(np.abs(f - 1.0) <= 0.01 + 1e-6) and np.ptp(f, axis=0).max() < 1e-6   # one factor per asset
    np.testing.assert_allclose(c1[1:] / c1[:-1], c0[1:] / c0[:-1], rtol=1e-6)         # returns unchanged
    np.testing.assert_allclose(p1[:, 1:, :], base[:, 1:, :], rtol=1e-5, atol=1e-5)    # close_norm, z-scores
    for k in range(4):
        ck = om.perturb_factor(9, k, 0.01)
        assert 0.99 <= ck <= 1.01
        # MACD / SMA / Bollinger scale with the price, RSI / CCI / DX do not
        for i, name in enumerate(om.INDICATORS):
            scaled = name in ("macd", "boll_ub", "boll_lb", "sma30", "sma60")
            ref = raw0[:, i, k] * (ck if scaled else 1.0)
            np.testing.assert_allclose(raw1[:, i, k], ref, rtol=1e-9, atol=1e-7)


# ------------------------------------------------------------- crypto market oracle (NEXT-3)
def test_vectorized_philox_matches_scalar():
    from oracle import philox
    rng = np.random.default_rng(3)
    ctr = rng.integers(0, 2**32, size=(200, 4), dtype=np.uint64)
    key = (0x9E3779B9, 0x0BADF00D)
    v = philox.philox4x32_10_np(ctr[:, 0], ctr[:, 1], ctr[:, 2], ctr[:, 3], *key)
    for i in range(200):
        assert tuple(int(x[i]) for x in v) == philox.philox4x32_10(tuple(int(c) for c in ctr[i]), key)


def test_crypto_generator_special_cases():
    """sigma = 0: the mid stays at m0 exactly; phi = 0: each factor is its innovation
    N(t, 7, k) exactly; row 0 holds f_0 = N(0, 7, k) and mid m0."""
    from oracle import crypto_market as ocm
    g = ocm.generate(40, 5, sigma=0.0, m0=123.5)
    assert np.all(g[:, 0] == np.float32(123.5))
    g = ocm.generate(12, 9, phi=0.0)
    for t in (0, 1, 7, 12):
        for k in (0, 3, 50, 100):
            assert g[t, 41 + k] == np.float32(ocm.normal(9, t, ocm.S_FACTOR, k))
    assert g[0, 0] == np.float32(5e4)


def test_crypto_generator_book_structure_and_sampled_rows():
    """Book invariants on every row (ask_0 > mid > bid_0, asks strictly increasing, bids
    strictly decreasing, sizes > 0, pad 0) and the element-wise full-length path equal to
    the plain loops on the rows they share."""
    from oracle import crypto_market as ocm
    g = ocm.generate(400, 41)
    mid, ask, bid = g[:, 0], g[:, 1:11], g[:, 21:31]
    assert np.all(ask[:, 0] > mid) and np.all(bid[:, 0] < mid)
    assert np.all(np.diff(ask, axis=1) > 0) and np.all(np.diff(bid, axis=1) < 0)
    assert np.all(g[:, 11:21] > 0) and np.all(g[:, 31:41] > 0) and np.all(g[:, 142:] == 0)
    rows = [0, 1, 2, 255, 256, 399, 400]
    assert np.array_equal(ocm.sampled_rows(400, 41, rows), g[rows])


def test_crypto_generator_distributions():
    """Moments of the drawn series against their definitions (3,000 steps): GBM log
    returns (drift -sigma^2/2, visible at sigma = 0.5; std sigma), lognormal spread and
    gaps (log-ratio mean 0, std 0.5), Exp(1) sizes, stationary AR(1) factors (variance 1,
    lag-1 autocorrelation phi)."""
    from oracle import crypto_market as ocm
    g = ocm.generate(1000, 77, sigma=0.5, m0=1e30).astype(np.float64)   # stays inside f32 range
    lr = np.diff(np.log(g[:, 0]))
    assert abs(lr.mean() - (-0.125)) < 4 * 0.5 / np.sqrt(1000) and abs(lr.std() - 0.5) < 0.04
    n = 3000
    g = ocm.generate(n, 78).astype(np.float64)
    lr = np.diff(np.log(g[:, 0]))
    assert abs(lr.std() - 1e-4) < 0.05e-4
    mid = g[:, 0]
    ls = np.log((g[:, 1] - mid) / (mid * 1e-4))
    assert abs(ls.mean()) < 0.05 and abs(ls.std() - 0.5) < 0.03
    lg = np.log(np.diff(g[:, 1:11], axis=1) / (mid[:, None] * 0.5e-4))
    assert abs(lg.mean()) < 0.03 and abs(lg.std() - 0.5) < 0.02
    sz = np.concatenate([g[:, 11:21].ravel(), g[:, 31:41].ravel()])
    assert abs(sz.mean() - 1.0) < 0.02 and abs(sz.std() - 1.0) < 0.03
    f = g[:, 41:142]
    assert abs(f.var(axis=0).mean() - 1.0) < 0.1
    ac = np.mean([np.corrcoef(f[:-1, k], f[1:, k])[0, 1] for k in range(101)])
    assert abs(ac - 0.9) < 0.02


# ---------------------------------------------------------------- stock OHLCV generator (R-SGEN)
from oracle import stock_market as osm  # noqa: E402


def test_stock_gen_sigma0_closed_form():
    """sigma = 0: the close is the deterministic GBM path S_{-1} e^{mu (d + 1)} (exact GBM step,
    dt = 1); high = max(open, close) and low = min(open, close) exactly (the |Z| terms vanish)."""
    D, K, mu = 40, 5, 3e-3
    x = osm.generate(D, K, seed=9, mu=mu, sigma=0.0)
    s_init = np.array([50.0 + 100.0 * osm.uniform(9, 0, osm.S_INIT, k) for k in range(K)])
    d = np.arange(D)[:, None]
    np.testing.assert_allclose(x[:, osm.CLOSE].astype(np.float64), s_init[None, :] * np.exp(mu * (d + 1)), rtol=3e-7)
    np.testing.assert_allclose(x[:, osm.OPEN].astype(np.float64), s_init[None, :] * np.exp(mu * d), rtol=3e-7)
    assert np.array_equal(x[:, osm.HIGH], np.maximum(x[:, osm.OPEN], x[:, osm.CLOSE]))
    assert np.array_equal(x[:, osm.LOW], np.minimum(x[:, osm.OPEN], x[:, osm.CLOSE]))


def test_stock_gen_flat_when_mu_sigma_zero():
    x = osm.generate(12, 3, seed=4, mu=0.0, sigma=0.0)
    for c in (osm.OPEN, osm.HIGH, osm.LOW, osm.CLOSE):
        assert np.array_equal(x[:, c], np.broadcast_to(x[0, osm.CLOSE], x[:, c].shape))


def test_stock_gen_bar_invariants_and_continuity():
    """S:36 bar invariants L <= min(O, C) <= max(O, C) <= H, positive prices and volumes; the
    open of day d is the close of day d - 1 (O_d = S_{d-1}, c.1); S0 in [50, 150)."""
    x = osm.generate(60, 6, seed=21)
    o, h, lo, c, v = (x[:, j] for j in range(5))
    assert np.all(lo <= np.minimum(o, c)) and np.all(np.maximum(o, c) <= h)
    assert np.all(lo > 0) and np.all(v > 0)
    assert np.array_equal(o[1:], c[:-1])
    assert np.all(o[0] >= 50.0 * (1 - 1e-6)) and np.all(o[0] < 150.0 * (1 + 1e-6))


def test_stock_gen_vectorised_equals_loops():
    """generate_np (element-wise Philox, for the C1 sizes) reproduces the plain loops: every
    value within one float32 ulp (NumPy's and libm's exp / log may differ in the last float64
    bit before the single f32 rounding)."""
    a = osm.generate(30, 7, seed=5)
    b = osm.generate_np(30, 7, seed=5)
    ulp = np.spacing(np.abs(a))
    assert np.all(np.abs(a.astype(np.float64) - b.astype(np.float64)) <= ulp)
    assert np.mean(a == b) > 0.99


def test_stock_gen_moments():
    """The drawn series have the distributions the generator states: daily log returns with
    mean mu - sigma^2 / 2 and std sigma (BASELINE configs[0]: GBM mu = 2e-4, sigma = 0.02 per
    day), the high / low excursions (0.5 sigma) |Z| with E|Z| = sqrt(2 / pi), log volumes with
    mean ln 1e6 and std 0.5; initial prices uniform on [50, 150)."""
    D, K, mu, sigma = 3000, 32, 2e-4, 0.02
    x = osm.generate_np(D, K, seed=77, mu=mu, sigma=sigma).astype(np.float64)
    o, h, lo, c, v = (x[:, j] for j in range(5))
    r = np.log(c[1:] / c[:-1]).ravel()
    n = r.size
    assert abs(r.mean() - (mu - 0.5 * sigma * sigma)) < 4 * sigma / math.sqrt(n)
    assert abs(r.std(ddof=1) / sigma - 1) < 0.03
    zh = (h / np.maximum(o, c) - 1) / (0.5 * sigma)
    zl = (1 - lo / np.minimum(o, c)) / (0.5 * sigma)
    for zz in (zh, zl):
        assert abs(zz.mean() / math.sqrt(2 / math.pi) - 1) < 0.03
    lv = np.log(v)
    assert abs(lv.mean() - math.log(1e6)) < 4 * 0.5 / math.sqrt(lv.size)
    assert abs(lv.std() / 0.5 - 1) < 0.03
    s0 = osm.generate_np(1, 4096, seed=3)[0, osm.OPEN].astype(np.float64)
    assert s0.min() >= 50.0 * (1 - 1e-6) and s0.max() < 150.0 * (1 + 1e-6)
    assert abs(s0.mean() - 100.0) < 4 * 100 / math.sqrt(12 * 4096)


def test_stock_gen_seeded():
    a = osm.generate(5, 3, seed=1)
    assert np.array_equal(a, osm.generate(5, 3, seed=1))
    assert not np.array_equal(a, osm.generate(5, 3, seed=2))
