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


# ------------------------------------------------------------- crypto market generation
def _close_f32(g, o):
    """Float64 on both sides, one f32 rounding each: equal up to 2 f32 ulps (the device's
    libm and chunked running sums differ from the oracle's in the last f64 bits, which
    can move a value across an f32 rounding boundary)."""
    g = g.astype(np.float64)
    o = o.astype(np.float64)
    tol = 2.0 * np.abs(o) * 2.0 ** -23 + 1e-30
    bad = np.abs(g - o) > tol
    assert not bad.any(), f"{int(bad.sum())} values beyond 2 ulp; first {np.argwhere(bad)[0].tolist()}"


def test_crypto_market_matches_oracle_small():
    """700 steps (three chunks of 256, the last ragged): every value against the oracle's
    plain loops."""
    import torch
    from oracle import crypto_market as ocm
    from paper_2501_10709_b200 import fin
    steps = 700
    rows = zeros((steps + 1, 144), torch.float32)
    fin.fin_crypto_market(steps, 41, rows)
    _close_f32(host(rows), ocm.generate(steps, 41))


def test_crypto_market_full_length_sampled():
    """BASELINE configs[3] length (480,000 steps): sampled rows (chunk edges, the ends)
    against the oracle's element-wise path; structural invariants on every row."""
    import torch
    from oracle import crypto_market as ocm
    from paper_2501_10709_b200 import fin
    steps = 480000
    rows = zeros((steps + 1, 144), torch.float32)
    fin.fin_crypto_market(steps, 43, rows)
    g = host(rows)
    sample = [0, 1, 255, 256, 257, 4097, 123457, 479999, 480000]
    _close_f32(g[sample], ocm.sampled_rows(steps, 43, sample))
    mid, ask, bid = g[:, 0], g[:, 1:11], g[:, 21:31]
    assert np.all(ask[:, 0] > mid) and np.all(bid[:, 0] < mid)
    assert np.all(np.diff(ask, axis=1) > 0) and np.all(np.diff(bid, axis=1) < 0)
    assert np.all(g[:, 11:21] > 0) and np.all(g[:, 142:] == 0)
    f = g[:, 41:142].astype(np.float64)
    assert abs(f.var(axis=0).mean() - 1.0) < 0.02


def test_crypto_market_rejects_bad_arguments():
    import torch
    from paper_2501_10709_b200 import fin
    rows = zeros((1, 144), torch.float32)
    with pytest.raises(Exception):
        fin.fin_crypto_market(0, 1, rows)
    rows = zeros((11, 144), torch.float32)
    with pytest.raises(Exception):
        fin.fin_crypto_market(10, 1, rows, phi=1.0)


# ---------------------------------------------------------------- stock OHLCV generation (R-SGEN)
def _within_ulps(g, o, n):
    g64, o64 = g.astype(np.float64), o.astype(np.float64)
    return np.all(np.abs(g64 - o64) <= n * np.spacing(np.abs(o).astype(np.float32)).astype(np.float64))


@pytest.mark.parametrize("D,K,seed,mu,sigma", [(120, 7, 3, 2e-4, 0.02), (50, 30, 11, 1e-3, 0.05), (9, 1, 2, 0.0, 0.0)])
def test_stock_market_matches_oracle_loops(D, K, seed, mu, sigma):
    """fin_stock_market against oracle/stock_market.generate (plain loops): every value within
    2 float32 ulps (float64 on both sides, device exp / log / sincos vs libm, one f32 rounding);
    the open of day d equals the close of day d - 1 bit for bit; bar invariants hold."""
    import torch
    from oracle import stock_market as osm
    from paper_2501_10709_b200 import fin
    x = zeros((D, 5, K), torch.float32)
    fin.fin_stock_market(D, K, seed, x, mu=mu, sigma=sigma)
    g = host(x)
    o = osm.generate(D, K, seed, mu=mu, sigma=sigma)
    assert _within_ulps(g, o, 2)
    assert np.array_equal(g[1:, osm.OPEN], g[:-1, osm.CLOSE])
    assert np.all(g[:, osm.LOW] <= np.minimum(g[:, osm.OPEN], g[:, osm.CLOSE]))
    assert np.all(np.maximum(g[:, osm.OPEN], g[:, osm.CLOSE]) <= g[:, osm.HIGH])


def test_stock_market_c1_size_and_chain():
    """The C1 shape (64 warm-up + 1008 stored days, 30 assets) against the oracle's
    element-wise path (all values within 2 f32 ulps), then the whole device pipeline:
    fin_stock_market -> fin_market_prepare -> fin_env_create -> a short fused rollout,
    the prepared tensor bit-identical to oracle/market.py on the GPU's own OHLCV (3 assets)."""
    import torch
    from oracle import stock_market as osm
    from paper_2501_10709_b200 import fin
    from synth import policy as spol
    D, K = sm.WARMUP_DAYS + 1008, 30
    x = zeros((D, 5, K), torch.float32)
    fin.fin_stock_market(D, K, 21, x)
    g = host(x)
    assert _within_ulps(g, osm.generate_np(D, K, 21), 2)
    ind = list(om.INDICATORS)
    mk = zeros((1008, 2 + len(ind), K), torch.float32)
    raw = zeros((len(ind), K, 1008), torch.float64)
    fin.fin_market_prepare(x, sm.WARMUP_DAYS, ind, mk, raw)
    o_mk, _ = om.prepare_stock_market(g[:, :, :3], sm.WARMUP_DAYS, ind)   # assets are independent: 3 of 30
    assert np.array_equal(host(mk)[:, :, :3], o_mk)
    cfg = fin.env_config(num_envs=300, num_assets=30, num_indicators=8, num_rows=1008, episode_len=30,
                         num_windows=195)
    env = fin.fin_env_create(cfg, host(mk))
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
    rew = zeros((40, 300), torch.float32)
    fin.fin_rollout(env, [pol], 40, fin.make_noise(fin.FIN_NOISE_PHILOX, 1), fin.make_traj(reward=rew))
    assert fin.fin_env_check(env) == 0 and np.isfinite(host(rew)).all()


def test_stock_market_rejects_bad_arguments():
    import torch
    from paper_2501_10709_b200 import fin
    x = zeros((10, 5, 4), torch.float32)
    for kw in (dict(sigma=-1.0), dict(s0_lo=0.0), dict(s0_lo=5.0, s0_hi=5.0), dict(mu=float("nan"))):
        with pytest.raises(fin.FinError):
            fin.fin_stock_market(10, 4, 1, x, **kw)
    with pytest.raises(ValueError):
        fin.fin_stock_market(10, 5, 1, x)
