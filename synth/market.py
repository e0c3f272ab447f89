"""Synthetic market data shaped like the paper's workloads.

Stock (BASELINE.json configs[0], configs[1]):
  close prices follow an exact-step geometric Brownian motion
  S_{d+1} = S_d * exp((mu - sigma^2/2) + sigma Z), S_0 ~ U(50,150), mu = 2e-4,
  sigma = 0.02 per day; OHLV is derived around the close; indicators are the
  paper's families (MACD, Bollinger bands, RSI, CCI, DX, SMA) with the
  parameters of DESIGN.md reading R11.  64 hidden warm-up days feed the
  indicators so no back-fill is needed (reading R12).

Stored stock layout (float32) ``market[d][c][k]``:
  c = 0            raw close (execution and marking price)
  c = 1            close / close[day 0]  (observation price, reading R13)
  c = 2 .. 2+I-1   indicators, z-scored per (asset, indicator) over the stored
                   days, computed in float64 then rounded once to float32.

Crypto (BASELINE.json configs[3]): mid GBM sigma = 1e-4 per step,
10-level book with lognormal half-spread and level gaps, Exp(1) sizes, 101
standard-normal AR(1) factors with phi = 0.9.  Row layout (144 float32):
  [mid, ask_px[10], ask_sz[10], bid_px[10], bid_sz[10], f[101], pad[2]].
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

WARMUP_DAYS = 64

STOCK_INDICATORS_C0 = ("macd", "rsi30", "cci30", "sma30")
STOCK_INDICATORS_C1 = ("macd", "boll_ub", "boll_lb", "rsi30", "cci30", "dx30", "sma30", "sma60")

CRYPTO_LEVELS = 10
CRYPTO_FACTORS = 101
CRYPTO_ROW = 144  # 1 + 4*10 + 101 + 2 pad (16-byte rows for TMA / vector loads)
CRYPTO_MID = 0
CRYPTO_ASK_PX = 1
CRYPTO_ASK_SZ = 11
CRYPTO_BID_PX = 21
CRYPTO_BID_SZ = 31
CRYPTO_F = 41


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


@dataclass
class StockMarket:
    close_all: np.ndarray      # [WARMUP + rows][K] float64 (hidden warm-up + stored)
    open_all: np.ndarray
    high_all: np.ndarray
    low_all: np.ndarray
    volume_all: np.ndarray
    indicators: tuple
    market: np.ndarray         # [rows][2+I][K] float32, the tensor both sides consume
    raw_indicators: np.ndarray = field(repr=False, default=None)  # [rows][I][K] f64 pre z-score

    @property
    def rows(self) -> int:
        return self.market.shape[0]

    @property
    def K(self) -> int:
        return self.market.shape[2]

    @property
    def I(self) -> int:
        return self.market.shape[1] - 2


# ---------------------------------------------------------------- GBM + bars
def gbm_close(n_days: int, K: int, rng: np.random.Generator, mu: float, sigma: float,
              s0: np.ndarray | None = None) -> np.ndarray:
    """Exact GBM step with dt = 1: S_{d+1} = S_d exp((mu - sigma^2/2) + sigma Z_d).

    Returns [n_days+1][K] float64 including S_0 at row 0.
    """
    if s0 is None:
        s0 = rng.uniform(50.0, 150.0, size=K)
    z = rng.standard_normal(size=(n_days, K))
    out = np.empty((n_days + 1, K), dtype=np.float64)
    out[0] = s0
    drift = mu - 0.5 * sigma * sigma
    for d in range(n_days):
        out[d + 1] = out[d] * np.exp(drift + sigma * z[d])
    return out


def ohlcv_from_close(path: np.ndarray, rng: np.random.Generator, sigma: float):
    """O_d = S_{d-1}; H_d = max(O,C)(1 + sigma/2 |Z_H|); L_d = min(O,C)(1 - sigma/2 |Z_L|);
    V_d ~ LogNormal(ln 1e6, 0.5).  ``path`` is [n+1][K] with S_{-1} at row 0."""
    close = path[1:]
    opn = path[:-1]
    zh = np.abs(rng.standard_normal(size=close.shape))
    zl = np.abs(rng.standard_normal(size=close.shape))
    high = np.maximum(opn, close) * (1.0 + 0.5 * sigma * zh)
    low = np.minimum(opn, close) * (1.0 - 0.5 * sigma * zl)
    vol = rng.lognormal(mean=np.log(1e6), sigma=0.5, size=close.shape)
    return opn, high, low, close, vol


# ---------------------------------------------------------------- indicators
def sma(x: np.ndarray, n: int) -> np.ndarray:
    """Simple moving average over the last n values (expanding before n)."""
    out = np.empty_like(x, dtype=np.float64)
    for d in range(x.shape[0]):
        lo = max(0, d - n + 1)
        out[d] = x[lo:d + 1].mean(axis=0)
    return out


def rolling_pstd(x: np.ndarray, n: int) -> np.ndarray:
    out = np.empty_like(x, dtype=np.float64)
    for d in range(x.shape[0]):
        lo = max(0, d - n + 1)
        out[d] = x[lo:d + 1].std(axis=0)
    return out


def ema(x: np.ndarray, alpha: float) -> np.ndarray:
    """EMA seeded at the first value: e_0 = x_0, e_d = e_{d-1} + alpha (x_d - e_{d-1})."""
    out = np.empty_like(x, dtype=np.float64)
    out[0] = x[0]
    for d in range(1, x.shape[0]):
        out[d] = out[d - 1] + alpha * (x[d] - out[d - 1])
    return out


def macd(close: np.ndarray) -> np.ndarray:
    return ema(close, 2.0 / 13.0) - ema(close, 2.0 / 27.0)


def rsi(close: np.ndarray, n: int = 30) -> np.ndarray:
    """Wilder RSI (alpha = 1/n), 100 when the average loss is 0, 50 on day 0."""
    out = np.empty_like(close, dtype=np.float64)
    out[0] = 50.0
    gain = np.zeros(close.shape[1])
    loss = np.zeros(close.shape[1])
    a = 1.0 / n
    for d in range(1, close.shape[0]):
        delta = close[d] - close[d - 1]
        g = np.maximum(delta, 0.0)
        l_ = np.maximum(-delta, 0.0)
        if d == 1:
            gain, loss = g, l_
        else:
            gain = gain + a * (g - gain)
            loss = loss + a * (l_ - loss)
        with np.errstate(divide="ignore", invalid="ignore"):
            rs = gain / loss
            val = 100.0 - 100.0 / (1.0 + rs)
        out[d] = np.where(loss == 0.0, 100.0, val)
    return out


def cci(high, low, close, n: int = 30) -> np.ndarray:
    """CCI = (TP - SMA_n(TP)) / (0.015 MAD_n(TP)); 0 when MAD = 0."""
    tp = (high + low + close) / 3.0
    out = np.empty_like(tp)
    for d in range(tp.shape[0]):
        lo = max(0, d - n + 1)
        w = tp[lo:d + 1]
        m = w.mean(axis=0)
        mad = np.abs(w - m).mean(axis=0)
        with np.errstate(divide="ignore", invalid="ignore"):
            v = (tp[d] - m) / (0.015 * mad)
        out[d] = np.where(mad == 0.0, 0.0, v)
    return out


def dx(high, low, close, n: int = 30) -> np.ndarray:
    """Wilder directional movement index DX = 100 |+DI - -DI| / (+DI + -DI)."""
    out = np.zeros_like(close)
    a = 1.0 / n
    sp = np.zeros(close.shape[1])
    sm = np.zeros(close.shape[1])
    st = np.zeros(close.shape[1])
    for d in range(1, close.shape[0]):
        up = high[d] - high[d - 1]
        dn = low[d - 1] - low[d]
        pdm = np.where((up > dn) & (up > 0), up, 0.0)
        mdm = np.where((dn > up) & (dn > 0), dn, 0.0)
        tr = np.maximum(high[d] - low[d],
                        np.maximum(np.abs(high[d] - close[d - 1]), np.abs(low[d] - close[d - 1])))
        if d == 1:
            sp, sm, st = pdm, mdm, tr
        else:
            sp = sp + a * (pdm - sp)
            sm = sm + a * (mdm - sm)
            st = st + a * (tr - st)
        with np.errstate(divide="ignore", invalid="ignore"):
            pdi = np.where(st > 0, 100.0 * sp / st, 0.0)
            mdi = np.where(st > 0, 100.0 * sm / st, 0.0)
            s = pdi + mdi
            out[d] = np.where(s > 0, 100.0 * np.abs(pdi - mdi) / s, 0.0)
    return out


def compute_indicator(name: str, o, h, l_, c) -> np.ndarray:
    if name == "macd":
        return macd(c)
    if name == "rsi30":
        return rsi(c, 30)
    if name == "cci30":
        return cci(h, l_, c, 30)
    if name == "sma30":
        return sma(c, 30)
    if name == "sma60":
        return sma(c, 60)
    if name == "dx30":
        return dx(h, l_, c, 30)
    if name in ("boll_ub", "boll_lb"):
        m = sma(c, 20)
        s = rolling_pstd(c, 20)
        return m + 2.0 * s if name == "boll_ub" else m - 2.0 * s
    raise ValueError(f"unknown indicator {name}")


def zscore(x: np.ndarray) -> np.ndarray:
    """Per-column z-score over axis 0 (population std); 0 where std = 0."""
    m = x.mean(axis=0)
    s = x.std(axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        z = (x - m) / s
    return np.where(s > 0, z, 0.0)


def stock_market(K: int, rows: int, indicators=STOCK_INDICATORS_C1, seed: int = 21,
                 mu: float = 2e-4, sigma: float = 0.02, warmup: int = WARMUP_DAYS) -> StockMarket:
    """Build the [rows][2+I][K] float32 stock market tensor (see module doc)."""
    rng = _rng(seed)
    n_days = warmup + rows
    path = gbm_close(n_days, K, rng, mu, sigma)
    o, h, l_, c, v = ohlcv_from_close(path, rng, sigma)
    raw = np.stack([compute_indicator(n, o, h, l_, c) for n in indicators], axis=1)  # [days][I][K]
    stored = slice(warmup, warmup + rows)
    raw_s = raw[stored]
    z = np.stack([zscore(raw_s[:, i, :]) for i in range(len(indicators))], axis=1)
    close_s = c[stored]
    market = np.empty((rows, 2 + len(indicators), K), dtype=np.float32)
    market[:, 0, :] = close_s.astype(np.float32)
    market[:, 1, :] = (close_s / close_s[0]).astype(np.float32)
    market[:, 2:, :] = z.astype(np.float32)
    return StockMarket(close_all=c, open_all=o, high_all=h, low_all=l_, volume_all=v,
                       indicators=tuple(indicators), market=market, raw_indicators=raw_s)


def stock_c0(seed: int = 11) -> StockMarket:
    """BASELINE.json configs[0]: K=4, I=4 (MACD, RSI-30, CCI-30, SMA-30), 65 stored days."""
    return stock_market(K=4, rows=65, indicators=STOCK_INDICATORS_C0, seed=seed)


def stock_c1(seed: int = 21, rows: int = 1008) -> StockMarket:
    """BASELINE.json configs[1]: K=30, I=8 (dim 301 = 1+30+30+240), 1008 GBM days."""
    return stock_market(K=30, rows=rows, indicators=STOCK_INDICATORS_C1, seed=seed)


# ---------------------------------------------------------------- crypto LOB
def crypto_market(steps: int, seed: int = 41, sigma: float = 1e-4, m0: float = 5e4,
                  phi: float = 0.9) -> np.ndarray:
    """[steps+1][144] float32 crypto rows (see module doc; constants are reading R28)."""
    from scipy.signal import lfilter

    rng = _rng(seed)
    n = steps + 1
    L = CRYPTO_LEVELS
    z = rng.standard_normal(size=n - 1)
    logm = np.empty(n)
    logm[0] = np.log(m0)
    logm[1:] = np.log(m0) + np.cumsum(-0.5 * sigma * sigma + sigma * z)
    mid = np.exp(logm)
    half = mid * 1e-4 * np.exp(0.5 * rng.standard_normal(size=n))
    gap_a = mid[:, None] * 0.5e-4 * np.exp(0.5 * rng.standard_normal(size=(n, L)))
    gap_b = mid[:, None] * 0.5e-4 * np.exp(0.5 * rng.standard_normal(size=(n, L)))
    ask = (mid + half)[:, None] + np.concatenate([np.zeros((n, 1)), np.cumsum(gap_a[:, :-1], axis=1)], axis=1)
    bid = (mid - half)[:, None] - np.concatenate([np.zeros((n, 1)), np.cumsum(gap_b[:, :-1], axis=1)], axis=1)
    ask_sz = rng.exponential(1.0, size=(n, L))
    bid_sz = rng.exponential(1.0, size=(n, L))
    f0 = rng.standard_normal(size=CRYPTO_FACTORS)
    eps = rng.standard_normal(size=(n, CRYPTO_FACTORS))
    eps[0] = f0 / np.sqrt(1.0 - phi * phi)  # so that f_0 = f0 after the filter gain below
    f = lfilter([np.sqrt(1.0 - phi * phi)], [1.0, -phi], eps, axis=0)
    rows = np.zeros((n, CRYPTO_ROW), dtype=np.float32)
    rows[:, CRYPTO_MID] = mid
    rows[:, CRYPTO_ASK_PX:CRYPTO_ASK_PX + L] = ask
    rows[:, CRYPTO_ASK_SZ:CRYPTO_ASK_SZ + L] = ask_sz
    rows[:, CRYPTO_BID_PX:CRYPTO_BID_PX + L] = bid
    rows[:, CRYPTO_BID_SZ:CRYPTO_BID_SZ + L] = bid_sz
    rows[:, CRYPTO_F:CRYPTO_F + CRYPTO_FACTORS] = f
    return rows
