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
