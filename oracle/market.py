"""Market preparation oracle (test infrastructure only).

The step before the rollout, written as plain per-asset loops in float64 in the order
the definitions state (no numpy reductions, so the operation order is explicit):

* per-asset price-scale perturbation (§5.1: "a random percentage change
  ranging from -1% to 1% ... applied to its prices, which shifts the price scale while
  preserving the original price trends"): c_k = 1 + m (2 u_k - 1), u_k the first
  Philox4x32-10 uniform of counter (k, 0, 0x4D4B5450, 0) under key = seed (reading
  R-PERTURB); open / high / low / close of asset k are multiplied by c_k, volume is not.
* the paper's indicator families with the parameters of reading R11:
  MACD = EMA12 - EMA26 (alpha = 2/(n+1), seeded at the first close); Bollinger bands
  SMA20 +- 2 population std over the last 20 closes; RSI-30 (Wilder, alpha = 1/30, 50 on
  day 0, 100 when the average loss is 0); CCI-30 = (TP - SMA30(TP)) / (0.015 MAD30(TP)),
  0 when MAD = 0; DX-30 (Wilder +DM / -DM / TR, alpha = 1/30); SMA-30, SMA-60.  Windows
  are expanding before they fill; the hidden warm-up days (reading R12) precede the
  stored rows.
* the stored tensor market[d][c][k] f32: c = 0 close, c = 1 close / close[first stored
  day], c = 2.. indicators z-scored per (asset, indicator) over the stored rows
  (two-pass population mean / std, 0 where std = 0), each rounded once to f32.
"""
from __future__ import annotations

import math

import numpy as np

from . import philox

INDICATORS = ("macd", "boll_ub", "boll_lb", "rsi30", "cci30", "dx30", "sma30", "sma60")
PERTURB_WORD = 0x4D4B5450   # "MKTP": counter word 2 of the perturbation draw


def perturb_factor(seed: int, k: int, magnitude: float) -> float:
    c = philox.philox4x32_10((k & 0xFFFFFFFF, 0, PERTURB_WORD, 0), (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))
    u = philox.uniform(c[0])
    return 1.0 + magnitude * (2.0 * u - 1.0)


def _window_mean(x, d, n):
    lo = max(0, d - n + 1)
    s = 0.0
    for j in range(lo, d + 1):
        s = s + x[j]
    return s / (d + 1 - lo)


def _window_pstd(x, d, n):
    lo = max(0, d - n + 1)
    m = _window_mean(x, d, n)
    s = 0.0
    for j in range(lo, d + 1):
        s = s + (x[j] - m) * (x[j] - m)
    return math.sqrt(s / (d + 1 - lo))


def ema(x, alpha):
    out = [x[0]]
    for d in range(1, len(x)):
        out.append(out[-1] + alpha * (x[d] - out[-1]))
    return out


def sma(x, n):
    return [_window_mean(x, d, n) for d in range(len(x))]


def macd(c):
    e12, e26 = ema(c, 2.0 / 13.0), ema(c, 2.0 / 27.0)
    return [a - b for a, b in zip(e12, e26)]


def bollinger(c, upper: bool, n: int = 20):
    out = []
    for d in range(len(c)):
        m = _window_mean(c, d, n)
        s = _window_pstd(c, d, n)
        out.append(m + 2.0 * s if upper else m - 2.0 * s)
    return out


def rsi(c, n: int = 30):
    a = 1.0 / n
    out = [50.0]
    gain = loss = 0.0
    for d in range(1, len(c)):
        delta = c[d] - c[d - 1]
        g = delta if delta > 0.0 else 0.0
        l_ = -delta if delta < 0.0 else 0.0
        if d == 1:
            gain, loss = g, l_
        else:
            gain = gain + a * (g - gain)
            loss = loss + a * (l_ - loss)
        out.append(100.0 if loss == 0.0 else 100.0 - 100.0 / (1.0 + gain / loss))
    return out


def cci(h, l_, c, n: int = 30):
    tp = [(h[d] + l_[d] + c[d]) / 3.0 for d in range(len(c))]
    out = []
    for d in range(len(tp)):
        lo = max(0, d - n + 1)
        m = _window_mean(tp, d, n)
        s = 0.0
        for j in range(lo, d + 1):
            s = s + abs(tp[j] - m)
        mad = s / (d + 1 - lo)
        out.append(0.0 if mad == 0.0 else (tp[d] - m) / (0.015 * mad))
    return out


def dx(h, l_, c, n: int = 30):
    a = 1.0 / n
    out = [0.0]
    sp = sm = st = 0.0
    for d in range(1, len(c)):
        up = h[d] - h[d - 1]
        dn = l_[d - 1] - l_[d]
        pdm = up if (up > dn and up > 0.0) else 0.0
        mdm = dn if (dn > up and dn > 0.0) else 0.0
        tr = max(h[d] - l_[d], max(abs(h[d] - c[d - 1]), abs(l_[d] - c[d - 1])))
        if d == 1:
            sp, sm, st = pdm, mdm, tr
        else:
            sp = sp + a * (pdm - sp)
            sm = sm + a * (mdm - sm)
            st = st + a * (tr - st)
        pdi = 100.0 * sp / st if st > 0.0 else 0.0
        mdi = 100.0 * sm / st if st > 0.0 else 0.0
        s = pdi + mdi
        out.append(100.0 * abs(pdi - mdi) / s if s > 0.0 else 0.0)
    return out


def indicator(name, h, l_, c):
    if name == "macd":
        return macd(c)
    if name == "boll_ub":
        return bollinger(c, True)
    if name == "boll_lb":
        return bollinger(c, False)
    if name == "rsi30":
        return rsi(c, 30)
    if name == "cci30":
        return cci(h, l_, c, 30)
    if name == "dx30":
        return dx(h, l_, c, 30)
    if name == "sma30":
        return sma(c, 30)
    if name == "sma60":
        return sma(c, 60)
    raise ValueError(name)


def zscore(x):
    n = len(x)
    s = 0.0
    for v in x:
        s = s + v
    m = s / n
    q = 0.0
    for v in x:
        q = q + (v - m) * (v - m)
    sd = math.sqrt(q / n)
    return [0.0 if sd == 0.0 else (v - m) / sd for v in x]


def prepare_stock_market(ohlcv, warmup: int, indicators=INDICATORS, magnitude: float = 0.0, seed: int = 0):
    """ohlcv f32 [D][5][K] (open, high, low, close, volume; D = warmup + rows), the first
    ``warmup`` days hidden -> market f32 [rows][2+I][K] and the raw stored indicators."""
    x = np.asarray(ohlcv, dtype=np.float64)
    D, _, K = x.shape
    rows = D - warmup
    I = len(indicators)
    market = np.zeros((rows, 2 + I, K), dtype=np.float32)
    raw = np.zeros((rows, I, K))
    for k in range(K):
        ck = perturb_factor(seed, k, magnitude)
        h = [float(x[d, 1, k]) * ck for d in range(D)]
        l_ = [float(x[d, 2, k]) * ck for d in range(D)]
        c = [float(x[d, 3, k]) * ck for d in range(D)]
        for d in range(rows):
            market[d, 0, k] = np.float32(c[warmup + d])
            market[d, 1, k] = np.float32(c[warmup + d] / c[warmup])
        for i, name in enumerate(indicators):
            series = indicator(name, h, l_, c)[warmup:]
            raw[:, i, k] = series
            market[:, 2 + i, k] = np.array(zscore(series), dtype=np.float32)
    return market, raw
