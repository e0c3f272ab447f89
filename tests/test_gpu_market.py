"""GPU parity of fin_market_prepare against oracle/market.py:
the f32 market tensor bit for bit (float64 in the definitions' order on both sides,
one rounding to f32), the raw indicator series bit for bit, with and without the
per-asset price-scale perturbation; and the prepared tensor drives an env exactly like
the host-built one."""
import numpy as np
import pytest

from gpu_util import dev, host, needs_gpu, zeros
from oracle import market as om
from synth import market as sm

pytestmark = [pytest.mark.gpu, needs_gpu]


def _ohlcv(K, rows, seed):
    m = sm.stock_market(K=K, rows=rows, seed=seed)
    x = np.stack([m.open_all, m.high_all, m.low_all, m.close_all, m.volume_all], axis=1).astype(np.float32)
    return m, x


@pytest.mark.parametrize("K,rows,mag,seed", [(4, 65, 0.0, 0), (30, 200, 0.01, 77), (7, 33, 0.05, 5)])
def test_market_prepare_bitwise(K, rows, mag, seed):
    import torch
    from paper_2501_10709_b200 import fin
    _, x = _ohlcv(K, rows, seed + 1)
    ind = list(om.INDICATORS)
    I = len(ind)
    mk = zeros((rows, 2 + I, K), torch.float32)
    raw = zeros((I, K, rows), torch.float64)
    fin.fin_market_prepare(dev(x), sm.WARMUP_DAYS, ind, mk, raw, magnitude=mag, seed=seed)
    o_mk, o_raw = om.prepare_stock_market(x, sm.WARMUP_DAYS, ind, magnitude=mag, seed=seed)
    assert np.array_equal(host(raw), np.transpose(o_raw, (1, 2, 0)))
    assert np.array_equal(host(mk), o_mk)


def test_market_prepare_c0_subset_and_env():
    """The C0 indicator subset (MACD, RSI-30, CCI-30, SMA-30) in that order, and an env
    created from the device-prepared tensor steps exactly like one from the oracle's."""
    import torch
    from paper_2501_10709_b200 import fin
    from gpu_util import stock_pair
    K, rows = 4, 65
    _, x = _ohlcv(K, rows, 11)
    ind = ["macd", "rsi30", "cci30", "sma30"]
    mk = zeros((rows, 6, K), torch.float32)
    raw = zeros((4, K, rows), torch.float64)
    fin.fin_market_prepare(dev(x), sm.WARMUP_DAYS, ind, mk, raw)
    o_mk, _ = om.prepare_stock_market(x, sm.WARMUP_DAYS, ind)
    assert np.array_equal(host(mk), o_mk)
    _, fcfg = stock_pair(num_envs=8, num_assets=4, num_indicators=4, num_rows=rows, episode_len=64, num_windows=1)
    envs = [fin.fin_env_create(fcfg, host(mk)), fin.fin_env_create(fcfg, o_mk)]
    acts = dev(np.random.default_rng(1).integers(-100, 101, (8, 4)).astype(np.int16))
    cash = [zeros(8, torch.float64) for _ in envs]
    for _ in range(5):
        for e in envs:
            fin.fin_env_step(e, acts)
    for e, c in zip(envs, cash):
        fin.fin_env_get_state(e, cash=c)
    assert np.array_equal(host(cash[0]), host(cash[1]))
