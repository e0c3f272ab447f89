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


# ---------------------------------------------------------------- policy-gradient step (R-PPO)
def test_ppo_grad_matches_oracle():
    """fin_ppo_grad against oracle.learn (ppo_head + mlp_backward) on the device forward's own
    outputs and hidden activations (teacher forced, as the layered MLP check): the C1 policy
    (301-256-256-30, Kaiming weights, random biases), 1,000 samples (ragged 64-row tiles), ratios
    spread across the clip range so both branches occur.  Every gradient tensor within
    2e-5 max|o| + 1e-4 |o| (fp32 contractions over 1,000 samples vs float64), the statistics to
    1e-9 (float64 head) and the clipped count exactly."""
    import torch
    from oracle import learn as olearn
    from oracle import mlp as omlp
    from paper_2501_10709_b200 import fin
    from synth import policy as spol
    rng = np.random.default_rng(21)
    dims = spol.STOCK_DIMS
    layers = spol.random_bias(spol.kaiming_bf16(dims, 3), 4)
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, layers)
    B = 1000
    xbits = spol.f64_to_bf16_bits(rng.standard_normal((B, dims[0])))
    z = torch.zeros((B, dims[-1]), dtype=torch.float32, device="cuda")
    hid = torch.zeros((B, 2, 256), dtype=torch.int16, device="cuda")
    xd = dev(xbits.view(np.int16))
    fin.fin_mlp_forward(pol, xd, z, hid)
    zg, hg = host(z).astype(np.float64), host(hid).view(np.uint16)
    a = (np.tanh(zg) + 0.1 * rng.standard_normal(zg.shape)).astype(np.float32)
    lp_true, _, _, _, _ = olearn.ppo_head(zg.tolist(), a.astype(np.float64).tolist(), [0.0] * B, [0.0] * B)
    logp_old = (np.array(lp_true) + rng.normal(0, 0.25, B)).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    L64 = omlp.layers_f64(layers)
    w2 = dev(L64[1][0].astype(np.float32))
    w3 = dev(L64[2][0].astype(np.float32))
    grads = [(zeros(w.shape, torch.float32), zeros(b.shape, torch.float32)) for w, b in L64]
    stats = zeros(4, torch.float64)
    fin.fin_ppo_grad(xd, hid, z, dev(a), dev(logp_old), dev(adv), w2, w3, grads, stats)
    _, rho, coef, g3, Lo = olearn.ppo_head(zg.tolist(), a.astype(np.float64).tolist(),
                                          logp_old.astype(np.float64).tolist(), adv.astype(np.float64).tolist())
    assert 0 < sum(c == 0.0 for c in coef) < B // 2
    xv = omlp.bf16_bits_to_f64(xbits)
    hv = omlp.bf16_bits_to_f64(hg)
    ref = olearn.mlp_backward_np(L64, xv, hv, g3)
    for (dw, db), (rw, rb) in zip(grads, ref):
        for g, o in ((host(dw).astype(np.float64), rw), (host(db).astype(np.float64), rb)):
            assert np.all(np.abs(g - o) <= 2e-5 * np.abs(o).max() + 1e-4 * np.abs(o)), float(np.abs(g - o).max())
    st = host(stats)
    assert st[0] == pytest.approx(Lo, rel=1e-9, abs=1e-12)
    assert st[1] == pytest.approx(np.mean(rho), rel=1e-9)
    assert round(st[2] * B) == sum(c == 0.0 for c in coef) and st[3] == B
    # the 1000-sample loops version of the oracle agrees with its vectorised restatement on a slice
    small = olearn.mlp_backward(L64, xv[:3].tolist(), hv[:3].tolist(), g3[:3])
    for (sw, sb), (rw, rb) in zip(small, olearn.mlp_backward_np(L64, xv[:3], hv[:3], g3[:3])):
        np.testing.assert_allclose(sw, rw, rtol=1e-10, atol=1e-14)


def test_adam_step_matches_oracle():
    import torch
    from oracle import learn as olearn
    from paper_2501_10709_b200 import fin
    rng = np.random.default_rng(5)
    n = 10007
    th, m, v, g = (rng.standard_normal(n) for _ in range(4))
    v = np.abs(v)
    dt, dm, dv = (dev(x.astype(np.float32)) for x in (th, m, v))
    fin.fin_adam_step(dt, dm, dv, dev(g.astype(np.float32)), 3, lr=1e-3)
    o_th, o_m, o_v = olearn.adam(th.astype(np.float32).astype(np.float64).tolist(),
                                 m.astype(np.float32).astype(np.float64).tolist(),
                                 v.astype(np.float32).astype(np.float64).tolist(),
                                 g.astype(np.float32).astype(np.float64).tolist(), 3, lr=1e-3)
    np.testing.assert_allclose(host(dm), o_m, rtol=2e-6, atol=1e-7)
    np.testing.assert_allclose(host(dv), o_v, rtol=2e-6, atol=1e-7)
    np.testing.assert_allclose(host(dt), o_th, rtol=2e-6, atol=2e-7)


def test_ppo_iteration_end_to_end():
    """One producer -> consumer iteration on the device: a fused rollout with Philox
    noise logs the env-private observation entries and market days; the learner rebuilds every
    sample's observation (bitwise the oracle's bf16 observation of the replayed state), the old
    policy's forward on it reproduces the rollout's network outputs bit for bit, the regenerated
    Philox noise reproduces the executed share counts, GAE gives the advantages, fin_ppo_prepare /
    fin_ppo_grad the gradient (ratio 1 at the old weights up to the f32 log pi_old; gradients against
    the oracle),
    Adam steps the float32 master weights, fin_policy_load installs them (the new forward passes
    the layered check against the oracle with the new bf16 weights; the surrogate at the new weights
    is finite -- its sign is not asserted: one Adam step moves every bf16 weight by about one
    rounding step, far outside the first-order regime of a sigma = 0.1 Gaussian), and the next
    rollout runs on the new policy."""
    import math

    import torch
    from gpu_util import stock_pair
    from oracle import learn as olearn
    from oracle import mlp as omlp
    from oracle import rollout as orol
    from oracle import stock as ostock
    from paper_2501_10709_b200 import fin
    from synth import market, policy as spol
    m = market.stock_c1(rows=150)
    N, T, K, seed = 300, 35, 30, 77
    ocfg, fcfg = stock_pair(num_envs=N, num_assets=K, num_indicators=8, num_rows=150, episode_len=30,
                            num_windows=20, window_block=128)
    env = fin.fin_env_create(fcfg, m.market)
    layers = spol.random_bias(spol.kaiming_bf16(spol.STOCK_DIMS, 7), 8)
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, layers)
    t_base = fin.fin_env_clock(env)
    logs = dict(actions=zeros((T, N, K), torch.int16), reward=zeros((T, N), torch.float32),
                done=zeros((T, N), torch.uint8), mlp_out=zeros((T, 1, N, K), torch.float32),
                obs_private=zeros((T, N, 32), torch.int16), day=zeros((T, N), torch.int32))
    fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_PHILOX, seed), fin.make_traj(**logs))
    assert fin.fin_env_clock(env) == t_base + T
    B = T * N
    idx = torch.arange(B, dtype=torch.int64, device="cuda")
    x = zeros((B, 301), torch.int16)
    fin.fin_gather_observations(env, logs["obs_private"], logs["day"], idx, x)
    xb = host(x).view(np.uint16).reshape(T, N, 301)
    # (a) the observations are the oracle's, bf16-quantised, on the replayed states
    acts = host(logs["actions"])
    st = ostock.reset(ocfg)
    for t in range(T):
        X = orol.stock_obs_batch(ocfg, st, m.market)
        assert np.array_equal(xb[t], spol.f64_to_bf16_bits(X)), t
        ostock.step(ocfg, st, m.market, acts[t])
    # (b) the old policy's forward reproduces the rollout's outputs bit for bit
    z_old = zeros((B, K), torch.float32)
    hid = zeros((B, 2, 256), torch.int16)
    fin.fin_mlp_forward(pol, x, z_old, hid)
    assert np.array_equal(host(z_old).reshape(T, N, K), host(logs["mlp_out"])[:, 0])
    # (c) the regenerated Philox noise reproduces the executed actions (up to .5 roundings)
    eps = zeros((B, K), torch.float32)
    fin.fin_rollout_noise(env, seed, t_base, idx, eps)
    zg, eg = host(z_old).astype(np.float64), host(eps).astype(np.float64)
    y = 100.0 * np.clip(np.tanh(zg) + 0.1 * eg, -1, 1)
    rha = np.sign(y) * np.floor(np.abs(y) + 0.5)
    bad = rha != acts.reshape(B, K)
    assert np.all(np.abs(np.abs(y[bad] - np.trunc(y[bad])) - 0.5) < 1e-4)
    # (d) advantages (no critic: V = 0) and the gradient at the old weights
    adv2 = zeros((T, N), torch.float32)
    ret = zeros((T, N), torch.float32)
    fin.fin_gae(logs["reward"], zeros((T + 1, N), torch.float32), logs["done"], adv2, ret, normalise=True)
    adv = adv2.reshape(B)
    a = zeros((B, K), torch.float32)
    logp_old = zeros(B, torch.float32)
    fin.fin_ppo_prepare(z_old, eps, a, logp_old)
    L64 = omlp.layers_f64(layers)
    w = [dev(W.astype(np.float32)) for W, _ in L64]
    b = [dev(bb.astype(np.float32)) for _, bb in L64]
    grads = [(zeros(W.shape, torch.float32), zeros(W.shape[0], torch.float32)) for W in w]
    stats = zeros(4, torch.float64)
    fin.fin_ppo_grad(x, hid, z_old, a, logp_old, adv, w[1], w[2], grads, stats)
    s0 = host(stats)
    # rho = 1 at the old weights, up to the f32 rounding of the stored log pi_old (~5e-6 of |log pi|)
    assert abs(s0[1] - 1.0) < 1e-5 and s0[2] == 0.0
    assert s0[0] == pytest.approx(float(host(adv).astype(np.float64).mean()), abs=1e-7)
    _, _, _, g3, _ = olearn.ppo_head(zg.tolist(), host(a).astype(np.float64).tolist(),
                                     host(logp_old).astype(np.float64).tolist(), host(adv).astype(np.float64).tolist())
    ref = olearn.mlp_backward_np(L64, omlp.bf16_bits_to_f64(xb.reshape(B, 301)),
                                 omlp.bf16_bits_to_f64(host(hid).view(np.uint16)), g3)
    for (dw, db), (rw, rb) in zip(grads, ref):
        for g, o in ((host(dw).astype(np.float64), rw), (host(db).astype(np.float64), rb)):
            assert np.all(np.abs(g - o) <= 5e-5 * np.abs(o).max() + 2e-4 * np.abs(o))
    # (e) Adam on the f32 master weights, install, check the new forward and the improvement
    params = w + b
    gl = [g for g, _ in grads] + [g for _, g in grads]
    for p, g in zip(params, gl):
        mm, vv = torch.zeros_like(p), torch.zeros_like(p)
        fin.fin_adam_step(p, mm, vv, g, 1, lr=1e-4)
    fin.fin_policy_load(pol, w, b)
    z_new = zeros((B, K), torch.float32)
    hid_new = zeros((B, 2, 256), torch.int16)
    fin.fin_mlp_forward(pol, x, z_new, hid_new)
    new_layers = [(spol.f64_to_bf16_bits(host(W).astype(np.float64)), host(bb)) for W, bb in zip(w, b)]
    N64 = omlp.layers_f64(new_layers)
    sub = slice(0, 2000)
    omlp.teacher_forced_layers(N64, omlp.bf16_bits_to_f64(xb.reshape(B, 301))[sub],
                               host(hid_new).view(np.uint16)[sub], host(z_new)[sub])
    fin.fin_ppo_grad(x, hid_new, z_new, a, logp_old, adv, dev(N64[1][0].astype(np.float32)),
                     dev(N64[2][0].astype(np.float32)), grads, stats)
    s1 = host(stats)
    assert math.isfinite(s1[0]) and math.isfinite(s1[1]) and s1[1] != s0[1]   # the policy moved
    assert not np.array_equal(host(z_new), host(z_old))
    # (f) the next rollout runs on the new policy (its z1s term recomputed for the new weights)
    fin.fin_rollout(env, [pol], 5, fin.make_noise(fin.FIN_NOISE_PHILOX, seed),
                    fin.make_traj(reward=zeros((5, N), torch.float32)))
    assert fin.fin_env_check(env) == 0


@pytest.mark.parametrize("variant", ["dqn", "double", "dueling"])
def test_dqn_grad_matches_oracle(variant):
    """fin_dqn_grad against oracle.learn (dqn_targets + dqn_head + mlp_backward) on the device
    forwards' own outputs (online net at s and s', a target net at s'): the C3 Q-net (103-128-128-3,
    dueling: -4), 1,000 transitions with 20% terminal ones; gradients within 2e-5 max|o| + 1e-4|o|,
    the loss and the mean target to 1e-6 (f32 network outputs, float64 head)."""
    import torch
    from oracle import learn as olearn
    from oracle import mlp as omlp
    from paper_2501_10709_b200 import fin
    from synth import policy as spol
    rng = np.random.default_rng(31)
    dueling = variant == "dueling"
    dims = tuple(spol.CRYPTO_DIMS[:-1]) + ((4,) if dueling else (3,))
    kind = fin.FIN_Q_DUELING if dueling else fin.FIN_Q_ARGMAX
    online = spol.random_bias(spol.kaiming_bf16(dims, 4), 5)
    target = spol.random_bias(spol.kaiming_bf16(dims, 6), 7)
    pol, tgt = fin.fin_policy_create(kind, online), fin.fin_policy_create(kind, target)
    B, O = 1000, dims[-1]
    xs = spol.f64_to_bf16_bits(rng.standard_normal((B, 103)))
    xn = spol.f64_to_bf16_bits(rng.standard_normal((B, 103)))

    def fwd(p, xb):
        z = zeros((B, O), torch.float32)
        h = zeros((B, 2, 128), torch.int16)
        fin.fin_mlp_forward(p, dev(xb.view(np.int16)), z, h)
        return z, h

    out, hid = fwd(pol, xs)
    qt, _ = fwd(tgt, xn)
    qo, _ = fwd(pol, xn) if variant == "double" else (None, None)
    act = rng.integers(0, 3, B).astype(np.uint8)
    rew = rng.standard_normal(B).astype(np.float32)
    done = (rng.random(B) < 0.2).astype(np.uint8)
    L64 = omlp.layers_f64(online)
    grads = [(zeros(W.shape, torch.float32), zeros(W.shape[0], torch.float32)) for W, _ in L64]
    stats = zeros(4, torch.float64)
    fin.fin_dqn_grad(dev(xs.view(np.int16)), hid, out, dev(act), dev(rew), dev(done), qt,
                     dev(L64[1][0].astype(np.float32)), dev(L64[2][0].astype(np.float32)), grads, stats,
                     q_next_online=qo, gamma=0.99, dueling=dueling)
    y = olearn.dqn_targets(host(qt).astype(np.float64).tolist(), rew.astype(np.float64), done, 0.99,
                           q_next_online=None if qo is None else host(qo).astype(np.float64).tolist(), dueling=dueling)
    Lo, g = olearn.dqn_head(host(out).astype(np.float64).tolist(), act, y, dueling)
    ref = olearn.mlp_backward_np(L64, omlp.bf16_bits_to_f64(xs), omlp.bf16_bits_to_f64(host(hid).view(np.uint16)), g)
    for (dw, db), (rw, rb) in zip(grads, ref):
        for gg, o in ((host(dw).astype(np.float64), rw), (host(db).astype(np.float64), rb)):
            assert np.all(np.abs(gg - o) <= 2e-5 * np.abs(o).max() + 1e-4 * np.abs(o)), float(np.abs(gg - o).max())
    st = host(stats)
    assert st[0] == pytest.approx(Lo, rel=1e-6) and st[2] == pytest.approx(np.mean(y), rel=1e-6, abs=1e-9)
    assert st[3] == B


@pytest.mark.parametrize("dims,kind", [((301, 256, 256, 30), 0), ((301, 64, 32, 30), 1), ((25, 128, 128, 4), 2),
                                       ((103, 128, 128, 3), 3), ((103, 128, 128, 4), 4),
                                       ((103, 128, 128, 128, 3), 3)])
def test_policy_load_equals_create(dims, kind):
    """fin_policy_load (the device gather into the tcgen05 image, bf16 round to nearest even, the
    factored nets' shared W1 columns, biases) installs exactly what fin_policy_create packs on the host
    from the same bf16 weights: the forward outputs and hidden activations are bit-identical, for every
    compiled network."""
    import torch
    from paper_2501_10709_b200 import fin
    from synth import policy as spol
    kinds = [fin.FIN_PPO_GAUSS, fin.FIN_SAC_SQUASH, fin.FIN_PPO_GAUSS, fin.FIN_Q_ARGMAX, fin.FIN_Q_DUELING]
    k = kinds[kind]
    target = spol.random_bias(spol.kaiming_bf16(dims, 31), 32)
    ref = fin.fin_policy_create(k, target)
    pol = fin.fin_policy_create(k, spol.random_bias(spol.kaiming_bf16(dims, 33), 34))
    # f32 master values that round to the target's bf16 (the bf16 value plus a sub-half-ulp offset)
    ws = []
    for w, _ in target:
        wf = (np.asarray(w, dtype=np.uint32) << 16).view(np.float32)
        ws.append(dev((wf * np.float32(1 + 2 ** -10)).astype(np.float32)))
    bs = [dev(np.asarray(b, dtype=np.float32)) for _, b in target]
    fin.fin_policy_load(pol, ws, bs)
    rng = np.random.default_rng(3)
    B = 300
    x = dev(spol.f64_to_bf16_bits(rng.standard_normal((B, dims[0]))).view(np.int16))
    H = max(dims[1:-1])
    outs = []
    for p in (ref, pol):
        z = zeros((B, dims[-1]), torch.float32)
        h = zeros((B, 2, H), torch.int16)
        fin.fin_mlp_forward(p, x, z, h)
        outs.append((host(z), host(h)))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
