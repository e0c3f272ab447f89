"""GPU parity of the consumer pieces: fin_gae bit-identical to
oracle/learn.gae before the f32 rounding (so the stored advantages and returns are equal
bit for bit), its batch normalisation within f32 rounding, and fin_kl_diversity against
the oracle's Eq. 5 term -- at small sizes in full and on the headline rollout's own
reward / done tensors (65,536 envs x 256 steps) on sampled envs."""
import numpy as np
import pytest

from gpu_util import dev, host, needs_gpu, zeros
from oracle import learn

pytestmark = [pytest.mark.gpu, needs_gpu]


def _inputs(T, N, seed, p_done=0.05):
    rng = np.random.default_rng(seed)
    r = rng.normal(0, 1, (T, N)).astype(np.float32)
    v = rng.normal(0, 2, (T + 1, N)).astype(np.float32)
    d = (rng.random((T, N)) < p_done).astype(np.uint8)
    return r, v, d


@pytest.mark.parametrize("T,N,gamma,lam", [(37, 300, 0.99, 0.95), (1, 1, 0.5, 0.0), (64, 129, 1.0, 1.0),
                                           (9, 1000, 0.0, 0.7), (37, 272, 0.99, 0.95), (3, 16, 0.9, 0.9)])
def test_gae_bitwise(T, N, gamma, lam):
    """N % 16 == 0 runs the TMA-staged kernel (272: a ragged last block of 16 envs; T = 37
    a ragged last row chunk), other N the register-prefetch kernel."""
    import torch
    from paper_2501_10709_b200 import fin
    r, v, d = _inputs(T, N, T + N)
    adv, ret = zeros((T, N), torch.float32), zeros((T, N), torch.float32)
    fin.fin_gae(dev(r), dev(v), dev(d), adv, ret, gamma=gamma, lam=lam)
    A, R = learn.gae(r.astype(np.float64), v.astype(np.float64), d, gamma, lam)
    assert np.array_equal(host(adv), np.array(A, dtype=np.float32))
    assert np.array_equal(host(ret), np.array(R, dtype=np.float32))


def test_gae_normalised():
    import torch
    from paper_2501_10709_b200 import fin
    T, N = 50, 784
    r, v, d = _inputs(T, N, 5)
    adv, ret = zeros((T, N), torch.float32), zeros((T, N), torch.float32)
    fin.fin_gae(dev(r), dev(v), dev(d), adv, ret, gamma=0.99, lam=0.95, normalise=True)
    A, R = learn.gae(r.astype(np.float64), v.astype(np.float64), d, 0.99, 0.95)
    An = np.array(learn.normalise(A))
    np.testing.assert_allclose(host(adv), An, rtol=1e-6, atol=1e-6)
    assert np.array_equal(host(ret), np.array(R, dtype=np.float32))


def test_gae_on_the_headline_rollout_sampled():
    """The bench's workload: a fused rollout's reward / done (65,536 envs, T = 256, resets
    every 30 steps), values from a seeded generator; 32 sampled envs against the oracle."""
    import torch
    from paper_2501_10709_b200 import fin
    from synth import market
    from synth import policy as spol
    m = market.stock_c1(rows=1008)
    N, T = 65536, 256
    cfg = fin.env_config(num_envs=N, num_assets=30, num_indicators=8, num_rows=1008, episode_len=30, num_windows=195)
    env = fin.fin_env_create(cfg, m.market)
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
    rew, done = zeros((T, N), torch.float32), zeros((T, N), torch.uint8)
    fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_PHILOX, 3), fin.make_traj(reward=rew, done=done))
    g = torch.Generator(device="cuda").manual_seed(9)
    val = torch.randn((T + 1, N), device="cuda", generator=g)
    adv, ret = zeros((T, N), torch.float32), zeros((T, N), torch.float32)
    fin.fin_gae(rew, val, done, adv, ret, gamma=0.99, lam=0.95)
    rng = np.random.default_rng(1)
    cols = sorted(set([0, N - 1] + list(rng.choice(N, 30, replace=False))))
    r, v, d = host(rew)[:, cols], host(val)[:, cols], host(done)[:, cols]
    A, R = learn.gae(r.astype(np.float64), v.astype(np.float64), d, 0.99, 0.95)
    assert np.array_equal(host(adv)[:, cols], np.array(A, dtype=np.float32))
    assert np.array_equal(host(ret)[:, cols], np.array(R, dtype=np.float32))
    assert host(done).sum() == N * (T // 30)


@pytest.mark.parametrize("kind,M,B,K", [(0, 3, 500, 30), (1, 3, 300, 3), (0, 15, 64, 30), (1, 1, 10, 3)])
def test_kl_diversity(kind, M, B, K):
    import torch
    from paper_2501_10709_b200 import fin
    rng = np.random.default_rng(M * B + K + kind)
    out = (np.tanh(rng.normal(size=(M, B, K))) if kind == 0 else rng.normal(size=(M, B, K))).astype(np.float32)
    D = zeros((M, M), torch.float64)
    fin.fin_kl_diversity(dev(out), D, kind=kind, sigma=0.1)
    ref = np.array(learn.kl_diversity(out.astype(np.float64).tolist(), 0.1, categorical=kind == 1))
    np.testing.assert_allclose(host(D), ref, rtol=1e-12, atol=1e-15)
