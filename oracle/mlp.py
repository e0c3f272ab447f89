"""Policy / Q network forward oracle (test infrastructure only).

BASELINE.json configs[1] (MLP 301-256-256-30, bf16 weights) and configs[3]
(103-128-128-3); PAPER.md P:134 (policy pi(.|s)), P:343-346 (feed-forward nets).
Reading R15: ReLU hidden activations; output layer linear (tanh / argmax are
applied by ``oracle.policy``).  q(.) = float64 -> bf16 RNE is applied exactly
where the GPU stores bf16: the observation and both hidden activations
(SURVEY §8(c) c.4).  Sums are float64.

  z1 = W1 q(x) + b1;  a1 = q(ReLU(z1));  z2 = W2 a1 + b2;  a2 = q(ReLU(z2));  z3 = W3 a2 + b3
"""
from __future__ import annotations

import numpy as np

from .quant import bf16_fast


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def layers_f64(layers):
    """[(W_bits uint16 [out][in], bias f32 [out])] -> [(W f64, b f64)] (exact widening)."""
    return [(bf16_bits_to_f64(w), np.asarray(b, dtype=np.float64)) for w, b in layers]


def forward(layers64, x: np.ndarray) -> np.ndarray:
    """Batched forward, x [B][in] float64 unquantised -> z_out [B][out] float64.

    The float64 matmul is a library primitive (``@``); ``forward_loops`` is the
    explicit-loop version it is pinned against.
    """
    h = bf16_fast(np.asarray(x, dtype=np.float64))
    n = len(layers64)
    for li, (w, b) in enumerate(layers64):
        z = h @ w.T + b
        if li < n - 1:
            h = bf16_fast(np.maximum(z, 0.0))
        else:
            h = z
    return h


FP32_ACC_BOUND = 2.0 ** -17   # reading R-TOL: fp32 accumulation error, relative to sum |w x|


def teacher_forced_layers(layers64, x, hidden_bits, z_dev, row_mask: bool = False):
    """Layer-by-layer check of a device forward pass (reading R-TOL).

    ``x`` [B][in] float64 unquantised observation (the oracle's own), ``hidden_bits``
    [B][2][H] uint16 bf16 bit patterns of the device's two hidden activations,
    ``z_dev`` [B][out] the device's output (or its first columns).  Each layer is recomputed in float64
    from the device's (bf16, exactly representable) input of that layer:
      z = W h_in + b,  delta = 2^-17 (|W| |h_in| + |b|)   (fp32-accumulation bound)
    * hidden: the device activation must equal bf16(ReLU(z)); where it does not, it
      must lie between bf16(ReLU(z - delta)) and bf16(ReLU(z + delta)) -- the bf16
      rounding of a pre-activation within the accumulation bound of a rounding
      boundary is ambiguous (both neighbours are correct); such cases are counted.
    * output: |z_dev - z| <= delta.
    Layer 1's input is q(x) computed by the oracle, so the observation encoding is
    checked bit-exactly through it.  Returns (n_ambiguous, n_hidden_total), plus with
    ``row_mask`` the [B] boolean mask of the rows that hold an ambiguous activation.
    """
    from .quant import bf16_fast
    h = bf16_fast(np.asarray(x, dtype=np.float64))
    hid = bf16_bits_to_f64(np.asarray(hidden_bits).view(np.uint16))
    n_amb = 0
    n_tot = 0
    rows = np.zeros(h.shape[0], dtype=bool)
    n = len(layers64)
    for li, (w, b) in enumerate(layers64):
        z = h @ w.T + b
        delta = FP32_ACC_BOUND * (np.abs(h) @ np.abs(w).T + np.abs(b)) + 1e-30
        if li < n - 1:
            dev = hid[:, li, : w.shape[0]]
            exp = bf16_fast(np.maximum(z, 0.0))
            diff = dev != exp
            if diff.any():
                lo = bf16_fast(np.maximum(z - delta, 0.0))
                hi = bf16_fast(np.maximum(z + delta, 0.0))
                ok = (dev >= lo) & (dev <= hi)
                bad = diff & ~ok
                assert not bad.any(), (
                    f"layer {li}: {int(bad.sum())} activations differ beyond the fp32 bound; first at "
                    f"{np.argwhere(bad)[0].tolist()}")
                n_amb += int(diff.sum())
                rows |= diff.any(axis=1)
            n_tot += dev.size
            h = dev          # teacher forcing: the next layer consumes the device's activations
        else:   # z_dev may hold the first c outputs only (a logged head)
            zd = np.asarray(z_dev, dtype=np.float64)
            c = zd.shape[-1]
            err = np.abs(zd - z[:, :c])
            bad = err > delta[:, :c]
            assert not bad.any(), f"output: {int(bad.sum())} beyond the fp32 bound, worst {float((err / delta).max()):.2f}x"
    if row_mask:
        return n_amb, n_tot, rows
    return n_amb, n_tot


def ambiguous_rows(layers64, x) -> np.ndarray:
    """[B] mask of the rows whose free-running float64 forward has a hidden pre-activation
    within the fp32 accumulation bound delta = 2^-17 (|W| |h| + |b|) of a bf16 rounding
    decision (bf16(ReLU(z - delta)) != bf16(ReLU(z + delta))): there a device that
    accumulates in fp32 may correctly round the other way (reading R-TOL), and the rest of
    that row's forward differs by one bf16 step of that activation.  For checks where the
    device's hidden activations are not logged."""
    h = bf16_fast(np.asarray(x, dtype=np.float64))
    rows = np.zeros(h.shape[0], dtype=bool)
    for w, b in layers64[:-1]:
        z = h @ w.T + b
        delta = FP32_ACC_BOUND * (np.abs(h) @ np.abs(w).T + np.abs(b)) + 1e-30
        lo = bf16_fast(np.maximum(z - delta, 0.0))
        hi = bf16_fast(np.maximum(z + delta, 0.0))
        rows |= (lo != hi).any(axis=1)
        h = bf16_fast(np.maximum(z, 0.0))
    return rows


def forward_loops(layers64, x) -> list:
    """Single-sample explicit-loop forward (pin for ``forward``)."""
    from .quant import bf16
    h = [bf16(float(v)) for v in x]
    n = len(layers64)
    for li, (w, b) in enumerate(layers64):
        out = []
        for j in range(w.shape[0]):
            s = 0.0
            for i in range(w.shape[1]):
                s = s + float(w[j, i]) * h[i]
            out.append(s + float(b[j]))
        if li < n - 1:
            h = [bf16(max(v, 0.0)) for v in out]
        else:
            h = out
    return h
