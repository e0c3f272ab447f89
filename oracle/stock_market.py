"""Stock OHLCV generation oracle (test infrastructure only).

The synthetic stand-in for the paper's DJIA-30 daily bars (the real data is
not available) with the distributions BASELINE.json configs[0] states: close
prices follow a geometric Brownian motion with S0 ~ U(50, 150), mu = 2e-4 and sigma = 0.02
per day, and OHLV "derived around the close".  The random numbers come
from the counter-based Philox4x32-10 generator keyed by the seed (reading R-SGEN), so the
device generator (fin_stock_market) and this oracle draw the same numbers:

  N(d, s, k) = component k % 4 of normals4(counter (d, s, k // 4, 0), key = seed)
               (float64 Box-Muller, oracle.philox.normals4)
  U(d, s, k) = ((x >> 8) + 0.5) 2^-24 of word k % 4 of Philox(counter (d, s, k // 4, 0))
  streams s: 11 initial price, 12 close, 13 high, 14 low, 15 volume (the crypto
             generator of R-CGEN uses 1..7)

For asset k and day d = 0 .. D-1 (row d of the [D][5][K] float32 tensor, channels open,
high, low, close, volume -- the layout fin_market_prepare takes):
  S_{-1} = lo + (hi - lo) U(0, 11, k);  l_{-1} = ln S_{-1}
  l_d = l_{d-1} + ((mu - (0.5 sigma) sigma) + sigma N(d, 12, k))      (exact GBM step, dt = 1)
  open_d = exp(l_{d-1}),  close_d = exp(l_d)                          (O_d = C_{d-1})
  high_d = max(open_d, close_d) (1 + (0.5 sigma) |N(d, 13, k)|)
  low_d  = min(open_d, close_d) (1 - (0.5 sigma) |N(d, 14, k)|)
  vol_d  = exp(ln 1e6 + 0.5 N(d, 15, k))                              (LogNormal(ln 1e6, 0.5))
Every value in float64 in this order, rounded once to float32; the running sum l_d is
accumulated left to right over d.
"""
from __future__ import annotations

import math

import numpy as np

from . import philox

S_INIT, S_CLOSE, S_HIGH, S_LOW, S_VOL = 11, 12, 13, 14, 15
OPEN, HIGH, LOW, CLOSE, VOLUME = 0, 1, 2, 3, 4


def _key(seed):
    return (seed & philox.MASK, (seed >> 32) & philox.MASK)


def normal(seed: int, d: int, s: int, k: int) -> float:
    return philox.normals4((d, s, k // 4, 0), seed)[k % 4]


def uniform(seed: int, d: int, s: int, k: int) -> float:
    return philox.uniform(philox.philox4x32_10((d, s, k // 4, 0), _key(seed))[k % 4])


def generate(D: int, K: int, seed: int, mu: float = 2e-4, sigma: float = 0.02, s0_lo: float = 50.0,
             s0_hi: float = 150.0) -> np.ndarray:
    """The [D][5][K] float32 OHLCV tensor with plain loops (small D, K only)."""
    out = np.zeros((D, 5, K), dtype=np.float32)
    drift = mu - (0.5 * sigma) * sigma
    hs = 0.5 * sigma
    lv0 = math.log(1e6)
    for k in range(K):
        lprev = math.log(s0_lo + (s0_hi - s0_lo) * uniform(seed, 0, S_INIT, k))
        for d in range(D):
            lcur = lprev + (drift + sigma * normal(seed, d, S_CLOSE, k))
            o = math.exp(lprev)
            c = math.exp(lcur)
            out[d, OPEN, k] = o
            out[d, HIGH, k] = max(o, c) * (1.0 + hs * abs(normal(seed, d, S_HIGH, k)))
            out[d, LOW, k] = min(o, c) * (1.0 - hs * abs(normal(seed, d, S_LOW, k)))
            out[d, CLOSE, k] = c
            out[d, VOLUME, k] = math.exp(lv0 + 0.5 * normal(seed, d, S_VOL, k))
            lprev = lcur
    return out


def _normals_np(seed: int, D: int, s: int, K: int) -> np.ndarray:
    """N(d, s, k) for all d < D, k < K -> [D][K] float64 (the element-wise Philox of
    oracle.philox, Box-Muller in float64 as oracle.philox.normals4)."""
    k0, k1 = _key(seed)
    nb = (K + 3) // 4
    d = np.arange(D, dtype=np.uint64)[:, None]
    b = np.arange(nb, dtype=np.uint64)[None, :]
    x = philox.philox4x32_10_np(d, s, b, 0, k0, k1)
    u = [((w >> np.uint64(8)).astype(np.float64) + 0.5) * 2.0 ** -24 for w in x]
    r0 = np.sqrt(-2.0 * np.log(u[0]))
    r1 = np.sqrt(-2.0 * np.log(u[2]))
    a0, a1 = 2.0 * math.pi * u[1], 2.0 * math.pi * u[3]
    z = np.stack([r0 * np.cos(a0), r0 * np.sin(a0), r1 * np.cos(a1), r1 * np.sin(a1)], axis=2)   # [D][nb][4]
    return z.reshape(D, nb * 4)[:, :K]


def generate_np(D: int, K: int, seed: int, mu: float = 2e-4, sigma: float = 0.02, s0_lo: float = 50.0,
                s0_hi: float = 150.0) -> np.ndarray:
    """``generate`` with the random draws made element-wise in NumPy (for the C1 sizes); the
    running sum is the same left-to-right loop over d (vectorised over assets)."""
    k0, k1 = _key(seed)
    nb = (K + 3) // 4
    w = philox.philox4x32_10_np(0, S_INIT, np.arange(nb, dtype=np.uint64), 0, k0, k1)
    u0 = np.stack([((x >> np.uint64(8)).astype(np.float64) + 0.5) * 2.0 ** -24 for x in w], axis=1).reshape(-1)[:K]
    drift = mu - (0.5 * sigma) * sigma
    hs = 0.5 * sigma
    zc, zh, zl, zv = (_normals_np(seed, D, s, K) for s in (S_CLOSE, S_HIGH, S_LOW, S_VOL))
    lp = np.empty((D + 1, K))
    lp[0] = np.log(s0_lo + (s0_hi - s0_lo) * u0)
    for d in range(D):
        lp[d + 1] = lp[d] + (drift + sigma * zc[d])
    o, c = np.exp(lp[:-1]), np.exp(lp[1:])
    out = np.empty((D, 5, K), dtype=np.float32)
    out[:, OPEN] = o
    out[:, HIGH] = np.maximum(o, c) * (1.0 + hs * np.abs(zh))
    out[:, LOW] = np.minimum(o, c) * (1.0 - hs * np.abs(zl))
    out[:, CLOSE] = c
    out[:, VOLUME] = np.exp(math.log(1e6) + 0.5 * zv)
    return out
