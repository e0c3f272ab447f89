"""Exact rounding helpers for the oracle (test infrastructure only).

* ``bf16(x)``  -- q(.) of DESIGN.md reading R14 / SURVEY §8(c) c.4: float64 -> bf16
  round-to-nearest-even, done exactly with ``fractions.Fraction`` (no float32
  intermediate), returned as the float64 value of the bf16 number.
* ``rha(x)``   -- round half away from zero (reading R18).
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


def bf16(x: float) -> float:
    """Value of the bf16 number nearest to float64 ``x`` (ties to even)."""
    if math.isnan(x):
        return math.nan
    if math.isinf(x) or x == 0.0:
        return x
    sign = -1.0 if x < 0 else 1.0
    a = Fraction(abs(x))
    # exponent e with 2^e <= a < 2^(e+1)
    e = math.frexp(abs(x))[1] - 1
    e = max(e, -126)              # below the normal range the spacing stays 2^-133
    ulp = Fraction(2) ** (e - 7)  # 7 fraction bits
    q, r = divmod(a, ulp)
    half = Fraction(1, 2)
    frac = r / ulp
    if frac > half or (frac == half and q % 2 == 1):
        q += 1
    val = q * ulp
    if val >= Fraction(2) ** 128:
        return sign * math.inf
    return sign * float(val)


def bf16_vec(xs) -> np.ndarray:
    return np.array([bf16(float(v)) for v in np.ravel(xs)], dtype=np.float64).reshape(np.shape(xs))


def rha(x: float) -> int:
    """Round half away from zero."""
    a = abs(x)
    n = math.floor(a)
    if a - n >= 0.5:      # a - n is exact for |x| < 2^52
        n += 1
    return n if x >= 0 else -n


def bf16_fast(x) -> np.ndarray:
    """Vectorised ``bf16`` for arrays (same result; pinned against ``bf16`` in the tests).

    For float64 ``x`` in the bf16 normal range, the two bf16 neighbours of ``x``
    are ``lo`` = x with the low 45 significand bits cleared (toward zero) and
    ``hi`` = lo + one bf16 ulp.  Both distances |x|-|lo| and |hi|-|x| are exact
    in float64 (same binade), so the nearest / ties-to-even choice is exact.
    Values outside the normal range fall back to the Fraction-based ``bf16``.
    """
    x = np.asarray(x, dtype=np.float64)
    flat = x.ravel()
    out = np.empty_like(flat)
    a = np.abs(flat)
    normal = (a >= 2.0 ** -126) & (a < (2.0 - 2.0 ** -8) * 2.0 ** 127)
    bits = a.view(np.uint64)
    mask = np.uint64((1 << 45) - 1)
    lo_bits = bits & ~mask
    lo = lo_bits.view(np.float64)
    hi = (lo_bits + np.uint64(1 << 45)).view(np.float64)
    dlo = a - lo
    dhi = hi - a
    lo_even = ((lo_bits >> np.uint64(45)) & np.uint64(1)) == 0
    pick_hi = (dhi < dlo) | ((dhi == dlo) & ~lo_even)
    r = np.where(pick_hi, hi, lo)
    out[normal] = np.copysign(r, flat)[normal]
    zero = flat == 0.0
    out[zero] = flat[zero]
    for i in np.nonzero(~normal & ~zero)[0]:
        out[i] = bf16(float(flat[i]))
    return out.reshape(x.shape)
