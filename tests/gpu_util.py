"""Helpers shared by the -m gpu parity tests: build matching oracle / library
configurations from one set of keyword arguments and move results to NumPy."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import stock as ostock

try:
    import torch
    HAVE_GPU = torch.cuda.is_available()
except Exception:  # pragma: no cover
    HAVE_GPU = False

needs_gpu = pytest.mark.skipif(not HAVE_GPU, reason="needs a CUDA device")

STOCK_KW = ("num_envs", "num_assets", "num_indicators", "num_rows", "episode_len", "window_stride",
            "window_offset", "num_windows", "window_block", "window_base", "advance_window_on_reset",
            "max_trade", "initial_cash", "cost_rate", "reward_scale", "autoreset", "env_offset")


def stock_pair(**kw):
    """(oracle StockEnvConfig, fin_env_config) built from the same keywords."""
    from paper_2501_10709_b200 import fin
    ocfg = ostock.StockEnvConfig(**{k: v for k, v in kw.items() if k in STOCK_KW})
    fkw = {k: (int(v) if isinstance(v, bool) else v) for k, v in kw.items()}
    fcfg = fin.env_config(task=fin.FIN_STOCK, **fkw)
    return ocfg, fcfg


def dev(x, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def zeros(shape, dtype):
    return torch.zeros(shape, dtype=dtype, device="cuda")


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def crypto_reward_tol(o_reward, pos_after, mid, mid_next, scale=1.0, fees=0.0):
    """SURVEY c.8's reward tolerance for the crypto env: 1e-5 |o| + 1e-5 S (|h'| |m' - m| + fees),
    h' the position after the trade (+-1 or 0)."""
    o = np.asarray(o_reward, dtype=np.float64)
    cond = np.abs(np.asarray(pos_after, dtype=np.float64)) * abs(float(mid_next) - float(mid)) + fees
    return 1e-5 * np.abs(o) + 1e-5 * scale * cond + 1e-30


def reward_tol(o_reward, o_hold, p, pn, scale=2.0 ** -12, cost_notional=None):
    """SURVEY c.8 reward tolerance: 1e-5 |o| + 1e-5 S (sum_k h'_k |p'_k - p_k| + fees)."""
    cond = np.abs(o_hold * np.abs(pn - p)).sum(axis=-1)
    if cost_notional is not None:
        cond = cond + cost_notional
    return 1e-5 * np.abs(o_reward) + 1e-5 * scale * cond + 1e-30
