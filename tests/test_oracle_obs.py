"""Pins for the oracle's observation functions (oracle/stock.py observation,
oracle/crypto.py observation) -- CPU only.

The GPU rollouts' layer-1 inputs are checked against these functions, so an
error here would be shared by both sides; each test below fixes them against
something other than the oracle: hand-typed vectors (tests/golden/
observation_cases.json) over a market whose entries name their own (day,
channel, asset), SPEC.md's encode_state examples and its D_s
formula.  A k-major feature order, h/100 in place of h/max_trade, an
off-by-one day, a wrong window mapping or a factor column shifted by one each
fail one of them.
"""
import numpy as np
import pytest

from oracle import crypto as ocry
from oracle import stock as ostock
from synth import market as smarket


def _coded_market(rows, K, I):
    """market[d][c][k] = 1000 d + 10 c + k + 0.5 (exact in fp32 for the sizes used)."""
    d = np.arange(rows, dtype=np.float64)[:, None, None]
    c = np.arange(2 + I, dtype=np.float64)[None, :, None]
    k = np.arange(K, dtype=np.float64)[None, None, :]
    m = (1000.0 * d + 10.0 * c + k + 0.5).astype(np.float32)
    assert np.array_equal(m.astype(np.float64), 1000.0 * d + 10.0 * c + k + 0.5)
    return m


def _stock_case(c):
    cfg = ostock.StockEnvConfig(**c["cfg"])
    m = _coded_market(cfg.num_rows, cfg.num_assets, cfg.num_indicators)
    st = ostock.reset(cfg)
    i = c["env"]
    st.cash[i] = c["cash"]
    st.hold[i] = list(c["hold"])
    st.t_ep[i] = c["t_ep"]
    return cfg, m, st, i


def test_stock_observation_hand_vectors(golden):
    for c in golden("observation_cases.json")["stock"]:
        cfg, m, st, i = _stock_case(c)
        x = ostock.observation(cfg, st, m, i)
        # exact: every entry is one correctly rounded division or an fp32 value widened exactly
        assert x == c["expect"], c["name"]
        # the day the entries name (1000 d + 10 + 0.5 for close_norm of asset 0)
        assert int(x[1] - 10.5) // 1000 == c["expect_day"], c["name"]
        assert len(x) == (cfg.num_indicators + 2) * cfg.num_assets + 1


def test_stock_observation_day_follows_the_steps(golden):
    """The day of the observation advances with the env's own steps: from reset,
    t zero-action steps later the entries are those of day start(w) + t (R10),
    with cash still b0 (1.0) and holdings 0."""
    c = next(c for c in golden("observation_cases.json")["stock"] if c["name"] == "test_window_offset30_global_id5")
    cfg = ostock.StockEnvConfig(**c["cfg"])
    m = _coded_market(cfg.num_rows, cfg.num_assets, cfg.num_indicators)
    st = ostock.reset(cfg)
    zero = np.zeros((cfg.num_envs, cfg.num_assets), dtype=np.int64)
    for t in range(c["t_ep"]):
        assert ostock.observation(cfg, st, m, 1) == [1.0, 1000.0 * (30 + t) + 10.5, 1000.0 * (30 + t) + 11.5,
                                                     0.0, 0.0, 1000.0 * (30 + t) + 20.5,
                                                     1000.0 * (30 + t) + 21.5, 1000.0 * (30 + t) + 30.5,
                                                     1000.0 * (30 + t) + 31.5]
        ostock.step(cfg, st, m, zero)
    x = ostock.observation(cfg, st, m, 1)
    assert x[1:3] == c["expect"][1:3] and x[5:] == c["expect"][5:]
    # env 0 has global id 4: w = (1 + 4 // 2) mod 3 = 0 as well -> same days
    assert ostock.observation(cfg, st, m, 0)[1] == x[1]


def test_stock_observation_spec_reset_example():
    """at reset the cash component is 1.0, holdings 0.0 and the price
    components 1.0 (prices divided by the first row's prices: window 0, day 0)."""
    mk = smarket.stock_c1(rows=40)
    cfg = ostock.StockEnvConfig(num_envs=3, num_assets=30, num_indicators=8, num_rows=40, episode_len=5,
                                num_windows=1)
    st = ostock.reset(cfg)
    for i in range(3):
        x = ostock.observation(cfg, st, mk.market, i)
        assert x[0] == 1.0
        assert x[1:31] == [1.0] * 30
        assert x[31:61] == [0.0] * 30
        assert len(x) == 301                       # BASELINE.json configs[1]: 1 + 30 + 30 + 30*8


@pytest.mark.parametrize("K,I,D", [(30, 7, 271), (30, 8, 301), (4, 4, 25)])
def test_stock_observation_dimension(K, I, D):
    """D_s = (I+2)K+1.  SPEC S:188's worked example prints 217 for
    K=30, I=7, but its own expression (7+2)*30+1 is 271 (a slip in SPEC; DESIGN.md
    reading R-DS): the formula binds, and BASELINE.json's 301 for I=8 agrees with it."""
    cfg = ostock.StockEnvConfig(num_envs=1, num_assets=K, num_indicators=I, num_rows=3, episode_len=1)
    m = np.ones((3, 2 + I, K), dtype=np.float32)
    assert len(ostock.observation(cfg, ostock.reset(cfg), m, 0)) == D


def test_stock_observation_is_pure(golden):
    """the same state twice -> identical rows."""
    c = golden("observation_cases.json")["stock"][0]
    cfg, m, st, i = _stock_case(c)
    assert ostock.observation(cfg, st, m, i) == ostock.observation(cfg, st, m, i)


def test_crypto_observation_hand_vectors(golden):
    rows = (100.0 * np.arange(8, dtype=np.float64)[:, None] + np.arange(144, dtype=np.float64)[None, :]
            + 0.25).astype(np.float32)
    for c in golden("observation_cases.json")["crypto"]:
        st = ocry.CryptoEnvState(cash=[1e6], pos=[c["pos"]], tau=[c["tau"]], t_ep=[c["t_ep"]])
        x = ocry.observation(st, rows, 0, c["max_hold"])
        assert len(x) == c["expect_len"], c["name"]
        assert x[:4] == c["expect_head"], c["name"]
        assert x[-1] == c["expect_last"], c["name"]
        # the 101 factors are the row's columns 41..141 in order
        assert x[2:] == [100.0 * c["t_ep"] + j + 0.25 for j in range(41, 142)], c["name"]
