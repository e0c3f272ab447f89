"""GPU parity of the env kernels (K1 step, K2 crypto step, K4 replay, state get/set)
against the float64 oracle, through the C ABI.  Integer holdings / done are
compared bit-exactly; cash and asset bit-exactly (the contract is rel 1e-5, the
kernels mirror the oracle's operation order so equality is expected); reward
(stored fp32) within SURVEY c.8's tolerance."""
import numpy as np
import pytest

from gpu_util import crypto_reward_tol, dev, host, needs_gpu, stock_pair, zeros
from oracle import crypto as ocry
from oracle import metrics as omet
from oracle import stock as ostock
from synth import inputs, market

pytestmark = [pytest.mark.gpu, needs_gpu]


def _fin():
    from paper_2501_10709_b200 import fin
    return fin


def _step_loop(fin, env, acts, K):
    import torch
    T, N = acts.shape[0], acts.shape[1]
    out = {k: [] for k in ("reward", "done", "cash", "hold", "asset", "actions")}
    for t in range(T):
        r, d, c = zeros(N, torch.float32), zeros(N, torch.uint8), zeros(N, torch.float64)
        h, a, ac = zeros((N, K), torch.int16), zeros(N, torch.float64), zeros((N, K), torch.int16)
        fin.fin_env_step(env, dev(acts[t], torch.int16),
                         fin.make_traj(reward=r, done=d, cash=c, hold=h, asset=a, actions=ac))
        for k, v in (("reward", r), ("done", d), ("cash", c), ("hold", h), ("asset", a), ("actions", ac)):
            out[k].append(host(v))
    return {k: np.stack(v) for k, v in out.items()}


def _compare_stock(g, o, mk, cfg):
    assert np.array_equal(g["hold"], o["hold"])
    assert np.array_equal(g["done"].astype(bool), o["done"])
    assert np.array_equal(g["cash"], o["cash"])            # bit-identical expected
    assert np.array_equal(g["asset"], o["asset"])
    np.testing.assert_allclose(g["cash"], o["cash"], rtol=1e-5, atol=1e-5)
    err = np.abs(g["reward"].astype(np.float64) - o["reward"])
    tol = 1e-5 * np.abs(o["reward"]) + 1e-5 * cfg.reward_scale * 1e4 + 1e-30
    assert np.all(err <= tol), float((err - tol).max())


def test_c0_step_parity():
    """BASELINE configs[0]: K=4, I=4, N=8, 64 steps, seeded integer actions."""
    import torch
    fin = _fin()
    m = market.stock_c0()
    ocfg, fcfg = stock_pair(num_envs=8, num_assets=4, num_indicators=4, num_rows=m.rows, episode_len=64)
    acts = inputs.stock_actions(64, 8, 4, seed=12)
    o, _ = ostock.run_actions(ocfg, m.market, acts)
    env = fin.fin_env_create(fcfg, m.market)
    g = _step_loop(fin, env, acts, 4)
    _compare_stock(g, o, m.market, ocfg)
    assert np.array_equal(g["actions"], acts)
    assert fin.fin_env_check(env) == 0


def test_c1_shape_step_parity_ragged_windows_resets():
    """C1 shapes (K=30, I=8) with N=300 (ragged vs 256-thread blocks), tile-aligned
    windows, auto-reset + test-mode window advance, actions beyond +-max_trade."""
    import torch
    fin = _fin()
    m = market.stock_c1(rows=120)
    kw = dict(num_envs=300, num_assets=30, num_indicators=8, num_rows=120, episode_len=7, window_stride=5,
              num_windows=15, window_block=128, advance_window_on_reset=True)
    ocfg, fcfg = stock_pair(**kw)
    acts = inputs.stock_actions(20, 300, 30, seed=7, max_trade=130)
    o, _ = ostock.run_actions(ocfg, m.market, acts)
    env = fin.fin_env_create(fcfg, m.market)
    g = _step_loop(fin, env, acts, 30)
    _compare_stock(g, o, m.market, ocfg)
    assert fin.fin_env_check(env) & fin.FIN_FLAG_ACTION_RANGE


def _redo_case(K=30, N=3000, cost=1e-3):
    """Envs whose cash sits exactly at, or one ulp around, the cost of q shares of one
    asset: cash = fl(q u) + {-1, 0, +1} ulp, u = fl(p (1 + c)), with dyadic and
    non-dyadic prices; each env asks for q + 3 shares of its asset, so the cash binds
    exactly at the affordability boundary of reading R5."""
    prices = np.array([0.75, 1.5, 64.0, 100.0, 0.1, 99.37, 33.3, 12.34, 250.5, 7.77] * 3, dtype=np.float32)[:K]
    mk = np.zeros((3, 3, K), dtype=np.float32)
    mk[:, 0, :] = prices[None, :]
    mk[:, 1, :] = 1.0
    u = prices.astype(np.float64) * (1.0 + cost)
    cash = np.empty(N)
    acts = np.zeros((N, K), dtype=np.int16)
    for i in range(N):
        k, q, v = i % K, 1 + (i // K) % 97, (i // (K * 97)) % 3 - 1
        b = q * u[k]
        cash[i] = np.nextafter(b, np.inf) if v > 0 else np.nextafter(b, -np.inf) if v < 0 else b
        acts[i, k] = q + 3
    return mk, cash, acts


@pytest.mark.parametrize("cost,K", [(1e-3, 30), (0.0, 30), (1e-3, 4)])
def test_exact_affordability_redo_path(cost, K):
    """The exact out-of-line buy path (env_stock.cuh stock_buys_exact, reached only when
    the fast floor estimate fails its check) runs -- the handle's event counter proves
    it -- and gives cash and holdings bitwise equal to the oracle's definition (R5), in
    K1 (fin_env_step) and K4 (fin_rollout_actions).  Control: unbinding buys never take it."""
    import torch
    fin = _fin()
    N = 3000
    mk, cash, acts = _redo_case(K, N, cost)
    ocfg, fcfg = stock_pair(num_envs=N, num_assets=K, num_indicators=1, num_rows=3, episode_len=2,
                            cost_rate=cost, window_block=N)
    p, pn = [float(x) for x in mk[0, 0]], [float(x) for x in mk[1, 0]]
    want_b, want_h = np.empty(N), np.zeros((N, K), dtype=np.int64)
    for i in range(N):
        b, h, _, _, _, _, _ = ostock.step_one(ocfg, float(cash[i]), [0] * K, p, pn, [int(x) for x in acts[i]])
        want_b[i], want_h[i] = b, h
    for path in ("k1", "k4"):
        env = fin.fin_env_create(fcfg, mk)
        fin.fin_env_set_state(env, cash=dev(cash), hold=zeros((N, K), torch.int16), t_ep=zeros(N, torch.int32))
        fin.fin_env_counters(env, clear=True)
        c, h = zeros((1, N), torch.float64), zeros((1, N, K), torch.int16)
        if path == "k1":
            fin.fin_env_step(env, dev(acts), fin.make_traj(cash=c, hold=h))
        else:
            fin.fin_rollout_actions(env, dev(acts[None]), 1, fin.make_traj(cash=c, hold=h))
        redo = fin.fin_env_counters(env)["exact_redo"]
        assert redo > 0, path
        assert np.array_equal(host(c)[0].view(np.uint64), want_b.view(np.uint64)), path
        assert np.array_equal(host(h)[0], want_h), path
        assert (want_b >= 0).all()
    # control: cash far from binding -> the fast path alone
    env = fin.fin_env_create(fcfg, mk)
    small = (acts > 0).astype(np.int16)
    c = zeros((1, N), torch.float64)
    fin.fin_env_step(env, dev(small), fin.make_traj(cash=c))
    assert fin.fin_env_counters(env)["exact_redo"] == 0


def test_exact_affordability_redo_path_fused_rollout():
    """The same boundary cases through the fused policy rollout (K3: the exact redo inline, the
    post-sell holdings kept in the tile's A operand): a zero-weight PPO policy (tanh 0 = 0) and
    supplied noise eps = (q + 3) / 10 on each env's asset give 100 clip(0.1 eps) = q + 3 shares; the
    redo counter proves the exact path ran, and cash / holdings equal the oracle's bit for bit."""
    import torch
    fin = _fin()
    K, N, I = 30, 3000, 8
    mk3, cash, acts = _redo_case(K, N, 1e-3)
    mk = np.zeros((3, 2 + I, K), dtype=np.float32)
    mk[:, :2, :] = mk3[:, :2, :]
    ocfg, fcfg = stock_pair(num_envs=N, num_assets=K, num_indicators=I, num_rows=3, episode_len=2, cost_rate=1e-3,
                            window_block=N)
    p, pn = [float(x) for x in mk[0, 0]], [float(x) for x in mk[1, 0]]
    want_b, want_h = np.empty(N), np.zeros((N, K), dtype=np.int64)
    for i in range(N):
        b, h, _, _, _, _, _ = ostock.step_one(ocfg, float(cash[i]), [0] * K, p, pn, [int(x) for x in acts[i]])
        want_b[i], want_h[i] = b, h
    dims = (1 + 2 * K + I * K, 256, 256, K)
    zero = [(np.zeros((o, i), dtype=np.uint16), np.zeros(o, dtype=np.float32)) for i, o in zip(dims[:-1], dims[1:])]
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, zero)
    env = fin.fin_env_create(fcfg, mk)
    fin.fin_env_set_state(env, cash=dev(cash), hold=zeros((N, K), torch.int16), t_ep=zeros(N, torch.int32))
    fin.fin_env_counters(env, clear=True)
    noise = (acts.astype(np.float32) / np.float32(10.0))[None, None]          # [T=1][M=1][N][K]
    c, h, a = zeros((1, N), torch.float64), zeros((1, N, K), torch.int16), zeros((1, N, K), torch.int16)
    fin.fin_rollout(env, [pol], 1, fin.make_noise(fin.FIN_NOISE_SUPPLIED, 0, dev(noise)),
                    fin.make_traj(cash=c, hold=h, actions=a))
    assert np.array_equal(host(a)[0], acts)
    assert fin.fin_env_counters(env)["exact_redo"] > 0
    assert np.array_equal(host(c)[0].view(np.uint64), want_b.view(np.uint64))
    assert np.array_equal(host(h)[0], want_h)


def test_replay_rollout_parity_and_episode_metrics():
    """K4: T steps in one launch; trajectory + online episode metrics vs oracle."""
    import torch
    fin = _fin()
    m = market.stock_c1(rows=200)
    N, T, K = 333, 40, 30
    kw = dict(num_envs=N, num_assets=K, num_indicators=8, num_rows=200, episode_len=9, window_stride=5,
              num_windows=30, window_block=64)
    ocfg, fcfg = stock_pair(**kw)
    acts = inputs.stock_actions(T, N, K, seed=9)
    o, _ = ostock.run_actions(ocfg, m.market, acts)
    env = fin.fin_env_create(fcfg, m.market)
    E = 8
    r, d = zeros((T, N), torch.float32), zeros((T, N), torch.uint8)
    c, h, a = zeros((T, N), torch.float64), zeros((T, N, K), torch.int16), zeros((T, N), torch.float64)
    em, ec, agg = zeros((E, N, 3), torch.float64), zeros(N, torch.int32), zeros(8, torch.float64)
    fin.fin_rollout_actions(env, dev(acts, torch.int16), T,
                            fin.make_traj(reward=r, done=d, cash=c, hold=h, asset=a, ep_metrics=em, ep_count=ec,
                                          agg=agg))
    g = {"reward": host(r), "done": host(d), "cash": host(c), "hold": host(h), "asset": host(a)}
    _compare_stock(g, o, m.market, ocfg)
    em, ec, agg = host(em), host(ec), host(agg)
    n_ep = 0
    cums = []
    for i in range(N):
        curves, _ = omet.split_episodes(1e6, o["asset"][:, i], o["done"][:, i])
        assert ec[i] == len(curves)
        for j, cv in enumerate(curves):
            cum, sh, mdd = omet.episode_metrics(cv)
            np.testing.assert_allclose(em[j, i, 0], cum, rtol=1e-9, atol=1e-15)
            np.testing.assert_allclose(em[j, i, 2], mdd, rtol=1e-9, atol=1e-15)
            if np.isnan(sh):
                assert np.isnan(em[j, i, 1])
            else:
                np.testing.assert_allclose(em[j, i, 1], sh, rtol=1e-7)
            cums.append(cum)
            n_ep += 1
    assert agg[fin.FIN_AGG_EPISODES] == n_ep
    np.testing.assert_allclose(agg[fin.FIN_AGG_SUM_CUM], np.sum(cums), rtol=1e-9)
    np.testing.assert_allclose(agg[fin.FIN_AGG_SUM_REWARD], np.sum(g["reward"].astype(np.float64)), rtol=1e-9)
    # state after the rollout equals the oracle's
    cs, hs, ts = zeros(N, torch.float64), zeros((N, K), torch.int16), zeros(N, torch.int32)
    fin.fin_env_get_state(env, cash=cs, hold=hs, t_ep=ts)
    ost = ostock.reset(ocfg)
    ostock.run_actions(ocfg, m.market, acts, ost)
    assert np.array_equal(host(cs), np.array(ost.cash)) and np.array_equal(host(hs), np.array(ost.hold))
    assert np.array_equal(host(ts), np.array(ost.t_ep))


def test_partition_invariance_two_handles():
    """S:216 / S:741: envs [0,N) in one handle == [0,a) and [a,N) in two handles (env_offset)."""
    import torch
    fin = _fin()
    m = market.stock_c1(rows=100)
    N, T, K = 260, 12, 30
    kw = dict(num_assets=K, num_indicators=8, num_rows=100, episode_len=5, num_windows=12, window_block=50,
              advance_window_on_reset=True)
    acts = inputs.stock_actions(T, N, K, seed=21)
    outs = []
    for lo, hi in ((0, N), (0, 117), (117, N)):
        _, fcfg = stock_pair(num_envs=hi - lo, env_offset=lo, **kw)
        env = fin.fin_env_create(fcfg, m.market)
        r, c = zeros((T, hi - lo), torch.float32), zeros((T, hi - lo), torch.float64)
        fin.fin_rollout_actions(env, dev(acts[:, lo:hi], torch.int16), T, fin.make_traj(reward=r, cash=c))
        outs.append((host(r), host(c)))
    assert np.array_equal(np.concatenate([outs[1][0], outs[2][0]], axis=1), outs[0][0])
    assert np.array_equal(np.concatenate([outs[1][1], outs[2][1]], axis=1), outs[0][1])


def test_set_state_teacher_forcing_and_no_autoreset_flag():
    import torch
    fin = _fin()
    m = market.stock_c0()
    N, K = 5, 4
    ocfg, fcfg = stock_pair(num_envs=N, num_assets=K, num_indicators=4, num_rows=m.rows, episode_len=3,
                            autoreset=False)
    env = fin.fin_env_create(fcfg, m.market)
    cash = np.array([10.0, 500.0, 1e6, 0.0, 123.456])
    hold = np.arange(N * K, dtype=np.int16).reshape(N, K)
    tep = np.array([0, 1, 2, 0, 1], dtype=np.int32)
    fin.fin_env_set_state(env, cash=dev(cash), hold=dev(hold), t_ep=dev(tep))
    st = ostock.reset(ocfg)
    st.cash, st.hold, st.t_ep = list(cash), [list(map(int, r)) for r in hold], list(map(int, tep))
    acts = inputs.stock_actions(4, N, K, seed=4)
    g = _step_loop(fin, env, acts[:1], K)
    o = ostock.step(ocfg, st, m.market, acts[0])
    assert np.array_equal(g["hold"][0], np.array(o["hold"])) and np.array_equal(g["cash"][0], np.array(o["cash"]))
    # env 2 finished its episode (t_ep 2 -> 3 = L); stepping it again raises the sticky flag
    _step_loop(fin, env, acts[1:2], K)
    assert fin.fin_env_check(env) & fin.FIN_FLAG_EPISODE_DONE


def test_create_rejects_bad_market():
    import pytest as _pt
    fin = _fin()
    m = market.stock_c0().market.copy()
    _, fcfg = stock_pair(num_envs=2, num_assets=4, num_indicators=4, num_rows=65, episode_len=64)
    bad = m.copy()
    bad[3, 0, 1] = -1.0
    with _pt.raises(fin.FinError) as e:
        fin.fin_env_create(fcfg, bad)
    assert e.value.code == fin.FIN_E_DATA
    bad = m.copy()
    bad[5, 3, 2] = np.nan
    with _pt.raises(fin.FinError):
        fin.fin_env_create(fcfg, bad)
    _, fcfg2 = stock_pair(num_envs=2, num_assets=4, num_indicators=4, num_rows=65, episode_len=65)
    with _pt.raises(fin.FinError) as e:
        fin.fin_env_create(fcfg2, m)
    assert e.value.code == fin.FIN_E_CONFIG


def test_crypto_step_parity():
    import torch
    fin = _fin()
    T, N = 300, 200
    rows = market.crypto_market(T, seed=41)
    ocfg = ocry.CryptoEnvConfig(num_envs=N, episode_len=T)
    fcfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=T + 1,
                          episode_len=T, reward_scale=1.0, cost_rate=0.0)
    env = fin.fin_env_create(fcfg, rows)
    rng = np.random.default_rng(3)
    st = ocry.reset(ocfg)
    for t in range(T):
        a = rng.integers(-1, 2, N)
        o = ocry.step(ocfg, st, rows, a)
        r, d, c, h, v = (zeros(N, torch.float32), zeros(N, torch.uint8), zeros(N, torch.float64),
                         zeros((N, 1), torch.int16), zeros(N, torch.float64))
        fin.fin_env_step(env, dev(a.reshape(N, 1), torch.int16), fin.make_traj(reward=r, done=d, cash=c, hold=h, asset=v))
        assert np.array_equal(host(h)[:, 0], np.array(o["pos"]))
        assert np.array_equal(host(c), np.array(o["cash"]))
        assert np.array_equal(host(v), np.array(o["asset"]))
        assert np.array_equal(host(d).astype(bool), np.array(o["done"]))
        err = np.abs(host(r).astype(np.float64) - np.array(o["reward"]))
        assert np.all(err <= crypto_reward_tol(o["reward"], o["pos"], rows[t, 0], rows[t + 1, 0])), t
    assert fin.fin_env_check(env) == 0


def _bench_cfg(fin, N):
    """The env of bench.py's HBM runs (C1 market, 1008 rows, 30-step episodes, 195 windows)."""
    kw = dict(num_envs=N, num_assets=30, num_indicators=8, num_rows=1008, episode_len=30, window_stride=5,
              num_windows=195, window_block=128)
    return stock_pair(**kw)


def _sample(N, n, seed):
    rng = np.random.default_rng(seed)
    return sorted(set([0, 127, 128, N - 1] + list(rng.choice(N, n, replace=False))))


def test_k1_bench_size_sampled():
    """K1 in the bench's launch configuration (N = 2^22 envs, persistent grid, TMA tile
    pipeline), 35 steps with a reset, fresh seeded actions every step: sampled envs
    (tile edges included) against the oracle run env by env -- holdings, done, cash
    bit-exact, reward within tolerance, final state."""
    import torch
    fin = _fin()
    N, T, K = 1 << 22, 35, 30
    m = market.stock_c1(rows=1008)
    ocfg, fcfg = _bench_cfg(fin, N)
    env = fin.fin_env_create(fcfg, m.market)
    cols = _sample(N, 40, 3)
    idx = torch.tensor(cols, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(11)
    acts, rew, done, cash = [], [], [], []
    for t in range(T):
        a = torch.randint(-100, 101, (N, K), device="cuda", generator=g, dtype=torch.int16)
        r, d, c = zeros(N, torch.float32), zeros(N, torch.uint8), zeros(N, torch.float64)
        fin.fin_env_step(env, a, fin.make_traj(reward=r, done=d, cash=c))
        acts.append(host(a[idx]))
        rew.append(host(r[idx])); done.append(host(d[idx])); cash.append(host(c[idx]))
    hold = zeros((N, K), torch.int16)
    fin.fin_env_get_state(env, hold=hold)
    hold = host(hold[idx])
    assert fin.fin_env_check(env) == 0
    acts, rew, done, cash = (np.stack(x) for x in (acts, rew, done, cash))
    for j, i in enumerate(cols):
        oc = ostock.StockEnvConfig(num_envs=1, env_offset=int(i), num_assets=30, num_indicators=8, num_rows=1008,
                                   episode_len=30, window_stride=5, num_windows=195, window_block=128)
        o, st = ostock.run_actions(oc, m.market, acts[:, j:j + 1])
        assert np.array_equal(o["done"][:, 0], done[:, j] > 0)
        assert np.array_equal(o["cash"][:, 0], cash[:, j])
        err = np.abs(rew[:, j].astype(np.float64) - o["reward"][:, 0])
        assert np.all(err <= 1e-5 * np.abs(o["reward"][:, 0]) + 1e-5 * 2.0 ** -12 * 1e4)
        assert np.array_equal(np.asarray(st.hold)[0], hold[j])


def test_k4_bench_size_sampled():
    """K4 replay in the bench's configuration (N = 2^20 envs, T = 32, actions [T][N][K]
    resident in HBM): sampled envs against the oracle."""
    import torch
    fin = _fin()
    N, T, K = 1 << 20, 32, 30
    m = market.stock_c1(rows=1008)
    ocfg, fcfg = _bench_cfg(fin, N)
    env = fin.fin_env_create(fcfg, m.market)
    g = torch.Generator(device="cuda").manual_seed(12)
    acts = torch.randint(-100, 101, (T, N, K), device="cuda", generator=g, dtype=torch.int16)
    rew, done = zeros((T, N), torch.float32), zeros((T, N), torch.uint8)
    fin.fin_rollout_actions(env, acts, T, fin.make_traj(reward=rew, done=done))
    assert fin.fin_env_check(env) == 0
    cols = _sample(N, 40, 4)
    idx = torch.tensor(cols, device="cuda")
    a, r, d = host(acts[:, idx]), host(rew[:, idx]), host(done[:, idx])
    cash = zeros(N, torch.float64)
    fin.fin_env_get_state(env, cash=cash)
    cash = host(cash[idx])
    for j, i in enumerate(cols):
        oc = ostock.StockEnvConfig(num_envs=1, env_offset=int(i), num_assets=30, num_indicators=8, num_rows=1008,
                                   episode_len=30, window_stride=5, num_windows=195, window_block=128)
        o, st = ostock.run_actions(oc, m.market, a[:, j:j + 1])
        assert np.array_equal(o["done"][:, 0], d[:, j] > 0)
        err = np.abs(r[:, j].astype(np.float64) - o["reward"][:, 0])
        assert np.all(err <= 1e-5 * np.abs(o["reward"][:, 0]) + 1e-5 * 2.0 ** -12 * 1e4)
        assert np.asarray(st.cash)[0] == cash[j]


@pytest.mark.parametrize("wblock", [1, 100])
def test_k1_k4_mixed_days_mispredicted_rows(wblock):
    """K1 and K4 (round-2 packed per-warp forms) where a warp's envs sit on different market days
    (window block 1: every env its own window) or the next slice's predicted day is wrong (window
    block 100 does not divide the slice distance): the warps take the L2 row-table path.  Several
    tiles per persistent block (N = 113,741: 889 tiles, a ragged last one), 33 steps with a reset
    and a test-mode window advance; sampled envs (slice and tile edges, the tail) against the oracle
    env by env -- holdings, done, cash bit-exact, reward within tolerance."""
    import torch
    fin = _fin()
    N, T, K = 444 * 128 * 2 + 77, 33, 30
    m = market.stock_c1(rows=1008)
    kw = dict(num_envs=N, num_assets=30, num_indicators=8, num_rows=1008, episode_len=30, window_stride=5,
              num_windows=195, window_block=wblock, advance_window_on_reset=True)
    ocfg, fcfg = stock_pair(**kw)
    cols = sorted(set(_sample(N, 30, 5 + wblock) + [31, 32, 63, 64, 95, 96, N - 77, N - 78]))
    idx = torch.tensor(cols, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(21 + wblock)
    acts = torch.randint(-100, 101, (T, N, K), device="cuda", generator=g, dtype=torch.int16)
    a = host(acts[:, idx])
    # K1: one fin_env_step per step
    env = fin.fin_env_create(fcfg, m.market)
    rew, done, cash = [], [], []
    for t in range(T):
        r, d, c = zeros(N, torch.float32), zeros(N, torch.uint8), zeros(N, torch.float64)
        fin.fin_env_step(env, acts[t], fin.make_traj(reward=r, done=d, cash=c))
        rew.append(host(r[idx])); done.append(host(d[idx])); cash.append(host(c[idx]))
    hold = zeros((N, K), torch.int16)
    fin.fin_env_get_state(env, hold=hold)
    hold = host(hold[idx])
    assert fin.fin_env_check(env) == 0
    rew, done, cash = (np.stack(x) for x in (rew, done, cash))
    # K4: the same actions replayed in one call on a fresh env
    env4 = fin.fin_env_create(fcfg, m.market)
    rew4, done4, cash4 = zeros((T, N), torch.float32), zeros((T, N), torch.uint8), zeros((T, N), torch.float64)
    fin.fin_rollout_actions(env4, acts, T, fin.make_traj(reward=rew4, done=done4, cash=cash4))
    assert fin.fin_env_check(env4) == 0
    rew4, done4, cash4 = host(rew4[:, idx]), host(done4[:, idx]), host(cash4[:, idx])
    for j, i in enumerate(cols):
        oc = ostock.StockEnvConfig(num_envs=1, env_offset=int(i), num_assets=30, num_indicators=8, num_rows=1008,
                                   episode_len=30, window_stride=5, num_windows=195, window_block=wblock,
                                   advance_window_on_reset=True)
        o, st = ostock.run_actions(oc, m.market, a[:, j:j + 1])
        tol = 1e-5 * np.abs(o["reward"][:, 0]) + 1e-5 * 2.0 ** -12 * 1e4
        for rr, dd, cc in ((rew, done, cash), (rew4, done4, cash4)):
            assert np.array_equal(o["done"][:, 0], dd[:, j] > 0), i
            assert np.array_equal(o["cash"][:, 0], cc[:, j]), i
            assert np.all(np.abs(rr[:, j].astype(np.float64) - o["reward"][:, 0]) <= tol), i
        assert np.array_equal(np.asarray(st.hold)[0], hold[j]), i


def test_k1_k4_extreme_cash_takes_the_exact_path():
    """Cash far beyond 2^32 shares of any asset (1e15, 2^40, +inf): the floor estimate's hi-word
    check fails, the exact redo runs (counter) and cash / holdings equal the oracle's definition
    bit for bit (R5: every buy is its full want), in K1 and K4, full tiles and a ragged one."""
    import torch
    fin = _fin()
    K = 30
    for N in (256, 300):
        mk = market.stock_c1(rows=80)
        ocfg, fcfg = stock_pair(num_envs=N, num_assets=K, num_indicators=8, num_rows=80, episode_len=5,
                                num_windows=10, window_block=N)
        acts = inputs.stock_actions(1, N, K, seed=3)[0]
        cash = np.array([[1e15, 2.0 ** 40, np.inf, 7.5e12][i % 4] for i in range(N)])
        st0 = ostock.reset(ocfg)
        st0.cash = [float(x) for x in cash]
        o = ostock.step(ocfg, st0, mk.market, acts)
        want_b, want_h = np.array(o["cash"]), np.array(o["hold"], dtype=np.int64)
        for path in ("k1", "k4"):
            env = fin.fin_env_create(fcfg, mk.market)
            fin.fin_env_set_state(env, cash=dev(cash), hold=zeros((N, K), torch.int16), t_ep=zeros(N, torch.int32))
            fin.fin_env_counters(env, clear=True)
            c, h = zeros((1, N), torch.float64), zeros((1, N, K), torch.int16)
            if path == "k1":
                fin.fin_env_step(env, dev(acts, torch.int16), fin.make_traj(cash=c, hold=h))
            else:
                fin.fin_rollout_actions(env, dev(acts[None], torch.int16), 1, fin.make_traj(cash=c, hold=h))
            assert fin.fin_env_counters(env)["exact_redo"] > 0, (path, N)
            assert np.array_equal(host(c)[0].view(np.uint64), want_b.view(np.uint64)), (path, N)
            assert np.array_equal(host(h)[0], want_h), (path, N)
