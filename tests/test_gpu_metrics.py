"""GPU parity of K6 (fin_episode_metrics: chunked segmented scans over a stored
equity log) against the oracle's per-episode two-pass metrics."""
import numpy as np
import pytest

from gpu_util import dev, host, needs_gpu, zeros
from oracle import metrics as omet

pytestmark = [pytest.mark.gpu, needs_gpu]


@pytest.mark.parametrize("T,N,p_done", [(64, 8, 0.05), (3000, 300, 0.01), (20000, 40, 0.0005), (7, 1, 0.5),
                                         (45, 270000, 1 / 30), (45, 262150, 1 / 30)])
def test_episode_metrics_parity(T, N, p_done):
    """Chunked three-pass scans (small N) and the single fused pass (N >= 2048 x 128:
    every row read once; checked on a seeded sample of 400 envs plus the first and
    last env) -- TMA-staged when N % 16 == 0 (270,000: a ragged last block of 48 envs,
    T = 45 a ragged last chunk of rows), register-prefetched otherwise (262,150)."""
    import torch
    from paper_2501_10709_b200 import fin
    rng = np.random.default_rng(T + N)
    eq = 1e6 * np.exp(np.cumsum(rng.normal(0, 0.01, (T + 1, N)), axis=0))
    done = rng.random((T, N)) < p_done
    done[-1, : N // 2] = True
    # after a done the next episode restarts from the reset equity (autoreset)
    E = int(done.sum(axis=0).max()) + 1
    em, ec, agg = zeros((E, N, 3), torch.float64), zeros(N, torch.int32), zeros(8, torch.float64)
    fin.fin_episode_metrics(dev(eq), dev(done.astype(np.uint8)), 1e6, 252.0, 0.0, em, ec, agg)
    em, ec, agg = host(em), host(ec), host(agg)
    n = 0
    sh_sum = 0.0
    full = N <= 1000
    check = range(N) if full else sorted(set([0, N - 1] + list(rng.choice(N, 400, replace=False))))
    for i in check:
        curves = []
        cur = [eq[0, i]]
        for t in range(T):
            cur.append(eq[t + 1, i])
            if done[t, i]:
                curves.append(cur)
                cur = [1e6]
        assert ec[i] == len(curves), i
        for j, cv in enumerate(curves):
            cum, sh, mdd = omet.episode_metrics(cv)
            np.testing.assert_allclose(em[j, i, 0], cum, rtol=1e-9, atol=1e-14)
            np.testing.assert_allclose(em[j, i, 2], mdd, rtol=1e-9, atol=1e-14)
            if np.isnan(sh):
                assert np.isnan(em[j, i, 1])
            else:
                np.testing.assert_allclose(em[j, i, 1], sh, rtol=1e-7, atol=1e-9)
                sh_sum += sh
            n += 1
    if full:
        assert agg[fin.FIN_AGG_EPISODES] == n
        np.testing.assert_allclose(agg[fin.FIN_AGG_SUM_SHARPE], sh_sum, rtol=1e-7, atol=1e-9)
    else:
        assert agg[fin.FIN_AGG_EPISODES] == ec.sum()


def test_episode_metrics_flat_equity():
    """A flat equity curve (zero actions) has zero returns: cum = MDD = 0 and
    Sharpe = NaN (std = 0, reading R21), on both fused-pass variants."""
    import torch
    from paper_2501_10709_b200 import fin
    for N in (262144, 262146):
        T = 60
        eq = torch.full((T + 1, N), 1e6, dtype=torch.float64, device="cuda")
        done = torch.zeros((T, N), dtype=torch.uint8, device="cuda")
        done[29::30] = 1
        em, ec = zeros((2, N, 3), torch.float64), zeros(N, torch.int32)
        fin.fin_episode_metrics(eq, done, 1e6, 252.0, 0.0, em, ec)
        em, ec = host(em), host(ec)
        assert (ec == 2).all()
        assert (em[:, :, 0] == 0).all() and (em[:, :, 2] == 0).all()
        assert np.isnan(em[:, :, 1]).all()


def test_episode_metrics_bench_size_sampled():
    """K6 in the bench's configuration (T = 2048, N = 2^18, lockstep 30-step episodes, the
    TMA-staged fused pass): sampled envs against the oracle's two-pass metrics."""
    import torch
    from paper_2501_10709_b200 import fin
    T, N = 2048, 1 << 18
    g = torch.Generator(device="cuda").manual_seed(5)
    done = torch.zeros((T, N), dtype=torch.uint8, device="cuda")
    done[29::30] = 1
    eq = 1e6 * torch.exp(torch.cumsum(0.01 * torch.randn((T + 1, N), device="cuda", generator=g,
                                                         dtype=torch.float64), 0))
    E = T // 30 + 1
    em, ec = zeros((E, N, 3), torch.float64), zeros(N, torch.int32)
    fin.fin_episode_metrics(eq, done, 1e6, 252.0, 0.0, em, ec)
    rng = np.random.default_rng(6)
    cols = sorted(set([0, 127, 128, N - 1] + list(rng.choice(N, 28, replace=False))))
    idx = torch.tensor(cols, device="cuda")
    e_h, d_h, em_h, ec_h = host(eq[:, idx]), host(done[:, idx]), host(em[:, idx]), host(ec[idx])
    for j in range(len(cols)):
        # episodes after the first restart from the reset equity 1e6
        curves = []
        cur = [float(e_h[0, j])]
        for t in range(T):
            cur.append(float(e_h[t + 1, j]))
            if d_h[t, j]:
                curves.append(cur)
                cur = [1e6]
        assert ec_h[j] == len(curves)
        for k, cv in enumerate(curves):
            cum, sh, mdd = omet.episode_metrics(cv)
            np.testing.assert_allclose(em_h[k, j], [cum, sh, mdd], rtol=1e-7, atol=1e-12)
