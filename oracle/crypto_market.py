"""Crypto market generation oracle (test infrastructure only).

The synthetic stand-in for the paper's BTC limit-order-book data (the
real data is not available) with the shapes and distributions of
BASELINE.json configs[3] (reading R28), drawn from the counter-based Philox4x32-10
generator so the device generator (fin_crypto_market) and this oracle draw the same
random numbers (reading R-CGEN):

  N(t, s, j) = component j % 4 of normals4(counter (t, s, j // 4, 0), key = seed)
               (Box-Muller in float64, oracle.philox.normals4)
  U(t, s, j) = ((x >> 8) + 0.5) 2^-24 of word j % 4 of Philox(counter (t, s, j // 4, 0))
  streams s: 1 mid, 2 half-spread, 3 ask gaps, 4 bid gaps, 5 ask sizes, 6 bid sizes,
             7 factors

Step t = 0 .. steps (row t of the [steps + 1][144] float32 tensor, layout of
synth.market: [mid, ask_px[10], ask_sz[10], bid_px[10], bid_sz[10], f[101], pad[2]]):
  log m_0 = ln m0;  log m_t = log m_{t-1} + ((-0.5 sigma) sigma + sigma N(t, 1, 0))
  m_t = exp(log m_t)                                         (GBM, sigma per step)
  h_t = m_t 1e-4 exp(0.5 N(t, 2, 0))                         (lognormal half-spread)
  ask_0 = m_t + h_t;  ask_l = ask_{l-1} + m_t 0.5e-4 exp(0.5 N(t, 3, l - 1))
  bid_0 = m_t - h_t;  bid_l = bid_{l-1} - m_t 0.5e-4 exp(0.5 N(t, 4, l - 1))
  ask_sz_l = -ln U(t, 5, l);  bid_sz_l = -ln U(t, 6, l)      (Exp(1) by inversion)
  f_{0,k} = N(0, 7, k);  f_{t,k} = phi f_{t-1,k} + sqrt(1 - phi^2) N(t, 7, k)
                                                             (stationary AR(1), 101 factors)
Every value in float64 in this order, rounded once to float32.
"""
from __future__ import annotations

import math

import numpy as np

from . import philox

LEVELS = 10
FACTORS = 101
ROW = 144
S_MID, S_HALF, S_ASK_GAP, S_BID_GAP, S_ASK_SZ, S_BID_SZ, S_FACTOR = 1, 2, 3, 4, 5, 6, 7


def _key(seed):
    return (seed & philox.MASK, (seed >> 32) & philox.MASK)


def normal(seed: int, t: int, s: int, j: int) -> float:
    return philox.normals4((t, s, j // 4, 0), seed)[j % 4]


def uniform(seed: int, t: int, s: int, j: int) -> float:
    return philox.uniform(philox.philox4x32_10((t, s, j // 4, 0), _key(seed))[j % 4])


def lob_row(seed: int, t: int, mid: float) -> list:
    """Columns 0 .. 40 of row t (mid, ask px / sz, bid px / sz) from the step's mid."""
    h = mid * 1e-4 * math.exp(0.5 * normal(seed, t, S_HALF, 0))
    ask, bid = [mid + h], [mid - h]
    for lv in range(1, LEVELS):
        ask.append(ask[-1] + mid * 0.5e-4 * math.exp(0.5 * normal(seed, t, S_ASK_GAP, lv - 1)))
        bid.append(bid[-1] - mid * 0.5e-4 * math.exp(0.5 * normal(seed, t, S_BID_GAP, lv - 1)))
    ask_sz = [-math.log(uniform(seed, t, S_ASK_SZ, lv)) for lv in range(LEVELS)]
    bid_sz = [-math.log(uniform(seed, t, S_BID_SZ, lv)) for lv in range(LEVELS)]
    return [mid] + ask + ask_sz + bid + bid_sz


def generate(steps: int, seed: int, sigma: float = 1e-4, m0: float = 5e4, phi: float = 0.9) -> np.ndarray:
    """The whole [steps + 1][144] float32 tensor with plain loops (small ``steps`` only)."""
    out = np.zeros((steps + 1, ROW), dtype=np.float32)
    drift = (-0.5 * sigma) * sigma
    gain = math.sqrt(1.0 - phi * phi)
    logm = math.log(m0)
    f = [normal(seed, 0, S_FACTOR, k) for k in range(FACTORS)]
    for t in range(steps + 1):
        if t > 0:
            logm = logm + (drift + sigma * normal(seed, t, S_MID, 0))
            f = [phi * f[k] + gain * normal(seed, t, S_FACTOR, k) for k in range(FACTORS)]
        out[t, :41] = lob_row(seed, t, math.exp(logm))
        out[t, 41:41 + FACTORS] = f
    return out


def _normals_np(seed: int, t: np.ndarray, s: int, blk: int) -> np.ndarray:
    """normals4 of counters (t, s, blk, 0) for an array of t -> [len(t)][4] float64."""
    k0, k1 = _key(seed)
    x = philox.philox4x32_10_np(t, s, blk, 0, k0, k1)
    u = [((w >> np.uint64(8)).astype(np.float64) + 0.5) * 2.0 ** -24 for w in x]
    r0 = np.sqrt(-2.0 * np.log(u[0]))
    r1 = np.sqrt(-2.0 * np.log(u[2]))
    a0, a1 = 2.0 * math.pi * u[1], 2.0 * math.pi * u[3]
    return np.stack([r0 * np.cos(a0), r0 * np.sin(a0), r1 * np.cos(a1), r1 * np.sin(a1)], axis=1)


def sampled_rows(steps: int, seed: int, rows, sigma: float = 1e-4, m0: float = 5e4, phi: float = 0.9) -> np.ndarray:
    """Rows ``rows`` of ``generate(steps, ...)`` for a large ``steps``: the same recurrences,
    with the random draws of all steps made by the element-wise Philox (library primitive:
    ``np.cumsum`` is the left-to-right running sum; the AR(1) loop runs over t in order)."""
    rows = sorted(int(r) for r in rows)
    last = rows[-1]
    t = np.arange(1, last + 1, dtype=np.uint64)
    drift = (-0.5 * sigma) * sigma
    z = _normals_np(seed, t, S_MID, 0)[:, 0]
    logm = np.concatenate([[math.log(m0)], math.log(m0) + np.cumsum(drift + sigma * z)])
    gain = math.sqrt(1.0 - phi * phi)
    nb = (FACTORS + 3) // 4
    eps = np.concatenate([_normals_np(seed, np.arange(0, last + 1, dtype=np.uint64), S_FACTOR, b)
                          for b in range(nb)], axis=1)[:, :FACTORS]
    f = eps[0].copy()
    want = set(rows)
    out = {}
    for tt in range(last + 1):
        if tt > 0:
            f = phi * f + gain * eps[tt]
        if tt in want:
            row = np.zeros(ROW, dtype=np.float32)
            row[:41] = lob_row(seed, tt, math.exp(logm[tt]))
            row[41:41 + FACTORS] = f
            out[tt] = row
    return np.stack([out[r] for r in rows])
