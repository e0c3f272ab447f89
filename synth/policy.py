"""Seeded policy / Q-network parameters (BASELINE.json configs[1..3]).

Kaiming-uniform with fan_in and gain sqrt(2): W ~ U(-sqrt(6/fan_in), +sqrt(6/fan_in))
drawn in float64 and rounded once to bf16 (round-to-nearest-even); biases 0
(reading R16).  Stored ``[out][in]`` unpadded; both sides read these bits.
bf16 is returned as its uint16 bit pattern so NumPy stays the only dependency.

Seeds (reading R16): C1 policy 0; C2 members 1, 2, 3; C3 Q-net 4.
"""
from __future__ import annotations

import numpy as np

STOCK_DIMS = (301, 256, 256, 30)
CRYPTO_DIMS = (103, 128, 128, 3)
# the paper's own networks (two hidden layers of 64 and 32 units;
# three 128-unit hidden layers), built as the NEXT-3 / NEXT-2 variants
STOCK_PAPER_DIMS = (301, 64, 32, 30)
CRYPTO_PAPER_DIMS = (103, 128, 128, 128, 3)


def f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float64 -> bf16 (RNE) exactly, via float64 arithmetic on the bit pattern.

    Rounds the float64 value directly (no intermediate float32 rounding), so
    there is no double-rounding.  Returns uint16 bit patterns.
    """
    x = np.asarray(x, dtype=np.float64)
    b = x.view(np.uint64)
    sign = (b >> np.uint64(63)).astype(np.uint16) << np.uint16(15)
    ax = np.abs(x)
    out = np.zeros(x.shape, dtype=np.uint16)
    # bf16: 8 exponent bits (bias 127), 7 fraction bits.  Work on |x| via frexp.
    with np.errstate(over="ignore", invalid="ignore"):
        m, e = np.frexp(ax)           # ax = m * 2^e, m in [0.5, 1)
    # normal range of bf16: exponent (e-1) in [-126, 127]
    ex = e - 1
    normal = (ax > 0) & np.isfinite(ax) & (ex >= -126)
    # significand scaled to 8 bits (1.xxxxxxx): s = m * 2^8 in [128, 256)
    s = m * 256.0
    r = np.where(normal, np.round(s), 0.0)  # np.round is half-to-even
    carry = r >= 256.0
    r = np.where(carry, r / 2.0, r)
    ex = np.where(carry, ex + 1, ex)
    frac = (r.astype(np.int64) - 128).astype(np.uint16)
    expo = (ex + 127).astype(np.int64)
    overflow = normal & (expo >= 255)
    nb = np.where(normal & ~overflow, (expo.clip(0, 254).astype(np.uint16) << np.uint16(7)) | frac, 0).astype(np.uint16)
    out = np.where(normal, nb, out)
    # subnormals of bf16: value = k * 2^-133, k in [0, 127]
    sub = (ax > 0) & np.isfinite(ax) & (ex < -126)
    k = np.where(sub, np.round(ax * 2.0 ** 133), 0.0)
    kb = k.astype(np.uint16)  # k == 128 rolls into the smallest normal bit pattern naturally
    out = np.where(sub, kb, out)
    inf_bits = np.uint16(0x7F80)
    out = np.where(np.isinf(ax) | overflow, inf_bits, out)
    out = np.where(np.isnan(x), np.uint16(0x7FC0), out)
    return (out | sign).astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def kaiming_bf16(dims, seed: int):
    """List of (W_bits [out][in] uint16, bias float32 [out]) per layer."""
    rng = np.random.Generator(np.random.PCG64(seed))
    layers = []
    for fan_in, fan_out in zip(dims[:-1], dims[1:]):
        bound = np.sqrt(6.0 / fan_in)
        w = rng.uniform(-bound, bound, size=(fan_out, fan_in))
        layers.append((f64_to_bf16_bits(w), np.zeros(fan_out, dtype=np.float32)))
    return layers


def random_bias(layers, seed: int, scale: float = 0.05):
    """Optional non-zero float32 biases for tests (biases are 0 in the configs)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return [(w, rng.uniform(-scale, scale, size=b.shape).astype(np.float32)) for w, b in layers]
