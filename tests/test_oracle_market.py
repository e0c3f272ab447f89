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
