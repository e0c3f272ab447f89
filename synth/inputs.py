"""Seeded per-step inputs: integer share actions and supplied Gaussian noise.

* ``stock_actions(T, N, K, seed)`` -- int16 U{-max_trade..max_trade}, shape [T][N][K]
  (BASELINE.json configs[0]: "seeded integer share deltas in [-100,100]").
* ``supplied_noise(T, M, N, K, seed)`` -- N(0,1) drawn in float64, stored float32,
  shape [T][M][N][K].  Parity mode feeds the same epsilon to both sides.
* ``crypto_uniforms`` -- float32 U[0,1) [T][N][2] for epsilon-greedy parity runs.
"""
from __future__ import annotations

import numpy as np


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def stock_actions(T: int, N: int, K: int, seed: int = 12, max_trade: int = 100) -> np.ndarray:
    return _rng(seed).integers(-max_trade, max_trade + 1, size=(T, N, K), dtype=np.int64).astype(np.int16)


def supplied_noise(T: int, M: int, N: int, K: int, seed: int = 23) -> np.ndarray:
    return _rng(seed).standard_normal(size=(T, M, N, K)).astype(np.float32)


def crypto_uniforms(T: int, N: int, seed: int = 43) -> np.ndarray:
    return _rng(seed).random(size=(T, N, 2)).astype(np.float32)
