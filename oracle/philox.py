"""Philox4x32-10 counter-based RNG + Box-Muller (test infrastructure only).

Production-mode noise of the rollout: both sides implement
the same counter-based generator (Salmon et al., SC'11, "Parallel random
numbers: as easy as 1, 2, 3"), keyed by the seed and countered by the GLOBAL
env id, so results do not depend on how envs are partitioned over GPUs.

  key     = (seed mod 2^32, seed >> 32)
  counter = (g, t_global, (member << 16) | block, 0)      stock noise, k in [4 block, 4 block + 4)
  counter = (g, t_global, 0xFFFF0000, 0)                  crypto epsilon-greedy draws
  u_i     = ((x_i >> 8) + 0.5) * 2^-24                     in (0, 1), exact in float32
  normals (z0, z1) = sqrt(-2 ln u0) (cos 2 pi u1, sin 2 pi u1), (z2, z3) likewise from (u2, u3)
"""
from __future__ import annotations

import math

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = (x & MASK for x in ctr)
    k0, k1 = key[0] & MASK, key[1] & MASK
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK
        hi1, lo1 = p1 >> 32, p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK, lo1, (hi0 ^ c3 ^ k1) & MASK, lo0
    return c0, c1, c2, c3


def uniform(x: int) -> float:
    return ((x >> 8) + 0.5) * 2.0 ** -24


def normals4(ctr, seed: int):
    x = philox4x32_10(ctr, (seed & MASK, (seed >> 32) & MASK))
    u = [uniform(v) for v in x]
    r0 = math.sqrt(-2.0 * math.log(u[0]))
    r1 = math.sqrt(-2.0 * math.log(u[2]))
    return (r0 * math.cos(2.0 * math.pi * u[1]), r0 * math.sin(2.0 * math.pi * u[1]),
            r1 * math.cos(2.0 * math.pi * u[3]), r1 * math.sin(2.0 * math.pi * u[3]))


def stock_noise(seed: int, g: int, t: int, member: int, K: int) -> list:
    out = []
    for blk in range((K + 3) // 4):
        out.extend(normals4((g, t, (member << 16) | blk, 0), seed))
    return out[:K]


def crypto_uniforms(seed: int, g: int, t: int):
    x = philox4x32_10((g, t, 0xFFFF0000, 0), (seed & MASK, (seed >> 32) & MASK))
    return uniform(x[0]), uniform(x[1])


def philox4x32_10_np(c0, c1, c2, c3, k0: int, k1: int):
    """The same Philox4x32-10 on NumPy arrays of counters (uint64 holding 32-bit values):
    the element-wise restatement of ``philox4x32_10`` for the full-length sampled checks
    (pinned against the scalar function and the known-answer vectors in the tests)."""
    import numpy as np
    m32 = np.uint64(MASK)
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & m32 for x in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0, k1 = k0 & MASK, k1 & MASK
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & m32
        hi1, lo1 = p1 >> np.uint64(32), p1 & m32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0)), lo1, (hi0 ^ c3 ^ np.uint64(k1)), lo0
    return c0, c1, c2, c3
