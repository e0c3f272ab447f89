"""Pins of oracle/learn.py (SURVEY §8(f) NEXT-4 consumer pieces): GAE against a worked
example, the SPEC special cases and the O(T^2) direct sum; batch
normalisation moments; the Eq. 5 KL term against closed forms and scipy's entropy."""
import math

import numpy as np
import pytest
from scipy.stats import entropy

from oracle import learn


def test_gae_worked_example():
    """T = 3, one env, gamma = 0.5, lambda = 0.5, done at t = 1 (by hand):
    V = [1, 2, 3, 4]; r = [1, 1, 1]
    t=2: delta = 1 + 0.5*4 - 3 = 0;            A2 = 0
    t=1: done -> delta = 1 - 2 = -1;           A1 = -1 (no carry across the done)
    t=0: delta = 1 + 0.5*2 - 1 = 1;            A0 = 1 + 0.25 * (-1) = 0.75"""
    A, R = learn.gae([[1.0], [1.0], [1.0]], [[1.0], [2.0], [3.0], [4.0]], [[0], [1], [0]], 0.5, 0.5)
    assert [a[0] for a in A] == [0.75, -1.0, 0.0]
    assert [r[0] for r in R] == [1.75, 1.0, 3.0]


def test_gae_lambda0_is_td_error_and_suffix_sums():
    rng = np.random.default_rng(1)
    T, N = 12, 5
    r = rng.normal(size=(T, N))
    v = rng.normal(size=(T + 1, N))
    d = rng.random((T, N)) < 0.2
    A, _ = learn.gae(r, v, d, 0.9, 0.0)
    td = r + 0.9 * v[1:] * (~d) - v[:-1]                    # lambda = 0: the one-step TD error
    np.testing.assert_allclose(A, td, rtol=0, atol=1e-14)
    A, _ = learn.gae(r, np.zeros((T + 1, N)), np.zeros((T, N), bool), 1.0, 1.0)
    np.testing.assert_allclose(A, np.cumsum(r[::-1], axis=0)[::-1], rtol=1e-13, atol=1e-13)


def test_gae_matches_direct_sum_and_all_done():
    rng = np.random.default_rng(2)
    T, N = 15, 6
    r, v, d = rng.normal(size=(T, N)), rng.normal(size=(T + 1, N)), rng.random((T, N)) < 0.25
    A, R = learn.gae(r, v, d, 0.97, 0.9)
    np.testing.assert_allclose(A, learn.gae_direct(r, v, d, 0.97, 0.9), rtol=0, atol=1e-10)
    np.testing.assert_allclose(np.array(R) - np.array(A), v[:-1], atol=1e-14)
    A, _ = learn.gae(r, v, np.ones((T, N), bool), 0.97, 0.9)
    np.testing.assert_array_equal(A, r - v[:-1])             # every step terminal: A = r - V


def test_normalise_moments():
    rng = np.random.default_rng(3)
    x = rng.normal(3.0, 2.0, size=(40, 7))
    y = np.array(learn.normalise(x.tolist()))
    assert abs(y.mean()) < 1e-12 and abs(y.std() - 1.0) < 1e-12
    z = np.array(learn.normalise([[2.5, 2.5], [2.5, 2.5]]))
    assert np.all(z == 0.0)


def test_kl_terms():
    # Gaussian: 1-D closed form (mu_j - mu_i)^2 / (2 sigma^2); identical members -> 0
    assert learn.kl_gaussian([0.3], [0.1], 0.1) == pytest.approx(0.04 / 0.02, rel=1e-14)
    assert learn.kl_gaussian([0.2, -0.5], [0.2, -0.5], 0.1) == 0.0
    # categorical against scipy's entropy(p, q) = sum p log(p / q)
    rng = np.random.default_rng(4)
    for _ in range(20):
        qj, qi = rng.normal(size=3), rng.normal(size=3)
        pj, pi = np.exp(qj) / np.exp(qj).sum(), np.exp(qi) / np.exp(qi).sum()
        assert learn.kl_categorical(list(qj), list(qi)) == pytest.approx(entropy(pj, pi), rel=1e-12, abs=1e-15)
    # D: zero diagonal, identical members -> 0, asymmetric for categorical
    out = rng.normal(size=(3, 5, 3)).tolist()
    D = np.array(learn.kl_diversity(out, 0.1, categorical=True))
    assert np.all(np.diag(D) == 0) and np.all(D[~np.eye(3, dtype=bool)] > 0)
    assert not np.allclose(D, D.T)
    same = [out[0], out[0]]
    assert np.all(np.array(learn.kl_diversity(same, 0.1)) == 0)
    G = np.array(learn.kl_diversity(out, 0.1))
    np.testing.assert_allclose(G, G.T, rtol=1e-12)            # equal-std Gaussians: symmetric


# ---------------------------------------------------------------- PPO / policy-gradient step (R-PPO)
def _tiny_net(rng, dims=(5, 6, 4, 3)):
    return [(rng.normal(0, 0.7, (o, i)), rng.normal(0, 0.1, o)) for i, o in zip(dims[:-1], dims[1:])]


def _forward64(layers, x):
    """Unquantised float64 forward of the 3-layer ReLU MLP: (z3, hidden [B][2][H])."""
    (w1, b1), (w2, b2), (w3, b3) = layers
    h1 = np.maximum(x @ w1.T + b1, 0.0)
    h2 = np.maximum(h1 @ w2.T + b2, 0.0)
    H = max(h1.shape[1], h2.shape[1])
    hid = np.zeros((x.shape[0], 2, H))
    hid[:, 0, :h1.shape[1]] = h1
    hid[:, 1, :h2.shape[1]] = h2
    return h2 @ w3.T + b3, hid


def _loss(layers, x, a, logp_old, adv):
    z3, _ = _forward64(layers, x)
    return -learn.ppo_head(z3.tolist(), a.tolist(), logp_old.tolist(), adv.tolist())[4]


def test_ppo_head_spec_examples():
    """rho = 1 everywhere -> the surrogate is the mean advantage; A > 0, rho = 2,
    clip 0.2 -> the sample contributes 1.2 A; zero advantages -> zero gradient; and the Gaussian
    log-density against its closed form at a = mu (the normalising constant only)."""
    z3 = [[0.3, -0.2], [0.0, 0.5]]
    mu = np.tanh(np.array(z3))
    a = (mu + 0.01).tolist()
    logp, _, _, _, _ = learn.ppo_head(z3, a, [0.0, 0.0], [0.0, 0.0])
    adv = [1.5, -0.5]
    _, rho, coef, g, L = learn.ppo_head(z3, a, logp, adv)
    assert rho == [1.0, 1.0] and L == pytest.approx(np.mean(adv), rel=1e-15)
    _, rho, _, _, L = learn.ppo_head(z3[:1], a[:1], [logp[0] - math.log(2.0)], [2.0])
    assert rho[0] == pytest.approx(2.0, rel=1e-14) and L == pytest.approx(1.2 * 2.0, rel=1e-14)
    _, _, coef, g, L = learn.ppo_head(z3, a, logp, [0.0, 0.0])
    assert L == 0.0 and np.all(np.array(g) == 0.0)
    lp, _, _, _, _ = learn.ppo_head([[0.2, 0.1, -0.3]], np.tanh([[0.2, 0.1, -0.3]]).tolist(), [0.0], [0.0])
    assert lp[0] == pytest.approx(-3 * math.log(0.1 * math.sqrt(2 * math.pi)), rel=1e-14)


def test_ppo_head_clipping_cases():
    """The clipped branch has zero gradient exactly when it is the minimum."""
    z3, a = [[0.1]], [[0.15]]
    lp, _, _, _, _ = learn.ppo_head(z3, a, [0.0], [0.0])
    for A, ratio, active in ((1.0, 1.5, False), (1.0, 0.5, True), (-1.0, 0.5, False), (-1.0, 1.5, True),
                             (1.0, 1.1, True), (-1.0, 0.9, True)):
        _, rho, coef, _, _ = learn.ppo_head(z3, a, [lp[0] - math.log(ratio)], [A])
        assert (coef[0] != 0.0) == active, (A, ratio)
        if active:
            assert coef[0] == pytest.approx(ratio * A, rel=1e-13)


def test_ppo_gradient_against_finite_differences():
    """d(-L)/dtheta from ppo_head + mlp_backward against central finite differences of the
    float64 loss, for every weight and bias of a small MLP, with a mix of clipped and unclipped
    samples; the vectorised backward equals the loops."""
    rng = np.random.default_rng(11)
    layers = _tiny_net(rng)
    B = 7
    x = rng.normal(size=(B, 5))
    z3, hid = _forward64(layers, x)
    a = np.tanh(z3) + 0.1 * rng.normal(size=z3.shape)
    logp_true, _, _, _, _ = learn.ppo_head(z3.tolist(), a.tolist(), [0.0] * B, [0.0] * B)
    logp_old = np.array(logp_true) + rng.normal(0, 0.3, B)      # ratios spread across the clip range
    adv = rng.normal(size=B)
    _, rho, coef, g3, _ = learn.ppo_head(z3.tolist(), a.tolist(), logp_old.tolist(), adv.tolist())
    assert any(c == 0.0 for c in coef) and any(c != 0.0 for c in coef)
    grads = learn.mlp_backward(layers, x.tolist(), hid.tolist(), g3)
    gnp = learn.mlp_backward_np(layers, x, hid, g3)
    for (dw, db), (dw2, db2) in zip(grads, gnp):
        np.testing.assert_allclose(dw, dw2, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(db, db2, rtol=1e-12, atol=1e-14)
    h = 1e-6
    for li in range(3):
        for which in (0, 1):
            p = layers[li][which]
            for idx in np.ndindex(p.shape):
                old = p[idx]
                p[idx] = old + h
                lp = _loss(layers, x, a, logp_old, adv)
                p[idx] = old - h
                lm = _loss(layers, x, a, logp_old, adv)
                p[idx] = old
                fd = (lp - lm) / (2 * h)
                an = grads[li][which][idx]
                assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd)), (li, which, idx, fd, an)


def test_adam_first_steps_closed_form():
    """Step 1: mhat = g, vhat = g^2, so theta moves by -lr g / (|g| + eps) (= -lr sign g for
    |g| >> eps); a zero gradient leaves theta; step 2 with the same g moves by the same amount."""
    g = [0.5, -2.0, 0.0, 1e-3]
    th, m, v = learn.adam([1.0, 1.0, 1.0, 1.0], [0.0] * 4, [0.0] * 4, g, 1, lr=0.1)
    for t, gi in zip(th, g):
        assert t == pytest.approx(1.0 - 0.1 * gi / (abs(gi) + 1e-8), rel=1e-12, abs=1e-15)
    th2, _, _ = learn.adam(th, m, v, g, 2, lr=0.1)
    for t2, t, gi in zip(th2, th, g):
        assert (t2 - t) == pytest.approx(-0.1 * gi / (abs(gi) + 1e-8), rel=1e-9, abs=1e-12)


# ---------------------------------------------------------------- DQN family (R-DQN)
def test_dqn_targets_spec_examples():
    """done = 1 -> y = r; gamma = 0 -> y = r; a constant target Q = c with r = 0,
    gamma = 0.99, done = 0 -> y = 0.99 c; Double DQN with online = target equals DQN; online argmax
    a1 while the target's max is at a2 -> the target's value at a1."""
    qt = [[1.0, 5.0, 2.0], [3.0, 3.0, 3.0]]
    assert learn.dqn_targets(qt, [0.5, -1.0], [1, 1], 0.99) == [0.5, -1.0]
    assert learn.dqn_targets(qt, [0.5, -1.0], [0, 0], 0.0) == [0.5, -1.0]
    assert learn.dqn_targets([[2.0, 2.0, 2.0]], [0.0], [0], 0.99) == [0.99 * 2.0]
    assert learn.dqn_targets(qt, [0.1, 0.2], [0, 0], 0.9, q_next_online=qt) == learn.dqn_targets(qt, [0.1, 0.2],
                                                                                                [0, 0], 0.9)
    y = learn.dqn_targets([[1.0, 5.0, 2.0]], [0.0], [0], 1.0, q_next_online=[[0.0, 1.0, 7.0]])
    assert y == [2.0]                                   # argmax online = 2 -> Q_target(s', 2)


def test_dueling_identities_and_head():
    """equal advantages -> Q = V for every action; V = 0, A = [1, 2, 3] ->
    Q = [-1, 0, 1]; argmax Q = argmax A.  The dueling head's output gradient sums to 2 (Q - y) / B
    on V and to 0 over the advantages (the mean-centering)."""
    assert learn.dueling_q([0.5, 0.5, 0.5, 2.0]) == [2.0, 2.0, 2.0]
    assert learn.dueling_q([1.0, 2.0, 3.0, 0.0]) == [-1.0, 0.0, 1.0]
    L, g = learn.dqn_head([[1.0, 2.0, 3.0, 0.5]], [2], [0.0], dueling=True)
    q = learn.dueling_q([1.0, 2.0, 3.0, 0.5])[2]
    assert L == q * q and g[0][3] == 2 * q and abs(sum(g[0][:3])) < 1e-15


def test_dqn_gradient_against_finite_differences():
    """d L / d theta (dqn_head + mlp_backward) against central finite differences, plain and dueling
    heads, with some terminal transitions; the target is held fixed (computed once)."""
    rng = np.random.default_rng(13)
    for dueling in (False, True):
        layers = _tiny_net(rng, (5, 6, 4, 4 if dueling else 3))
        B = 6
        x = rng.normal(size=(B, 5))
        xn = rng.normal(size=(B, 5))
        a = rng.integers(0, 3, B)
        r = rng.normal(size=B)
        done = rng.random(B) < 0.3
        qt, _ = _forward64(layers, xn)
        y = learn.dqn_targets(qt.tolist(), r, done, 0.9, dueling=dueling)

        def loss():
            out, _ = _forward64(layers, x)
            return learn.dqn_head(out.tolist(), a, y, dueling)[0]

        out, hid = _forward64(layers, x)
        _, g = learn.dqn_head(out.tolist(), a, y, dueling)
        grads = learn.mlp_backward(layers, x.tolist(), hid.tolist(), g)
        h = 1e-6
        for li in range(3):
            for which in (0, 1):
                p = layers[li][which]
                for idx in np.ndindex(p.shape):
                    old = p[idx]
                    p[idx] = old + h
                    lp = loss()
                    p[idx] = old - h
                    lm = loss()
                    p[idx] = old
                    fd = (lp - lm) / (2 * h)
                    assert abs(fd - grads[li][which][idx]) <= 1e-6 * max(1.0, abs(fd)), (dueling, li, which, idx)


# ---------------------------------------------------------------- actor-critic (R-AC)
def test_log1m_tanh2_stable_form():
    """ln(1 - tanh(u)^2) against the naive formula where it is accurate, and its asymptote
    2 (ln 2 - |u|) where tanh rounds to 1 (the naive form gives -inf there); even in u."""
    for u in np.linspace(-5, 5, 41):
        assert learn.log1m_tanh2(u) == pytest.approx(math.log(1.0 - math.tanh(u) ** 2), rel=1e-9, abs=1e-12)
        assert learn.log1m_tanh2(u) == pytest.approx(learn.log1m_tanh2(-u), rel=1e-13, abs=1e-15)
    for u in (30.0, -40.0, 300.0):
        assert learn.log1m_tanh2(u) == pytest.approx(2.0 * (math.log(2.0) - abs(u)), rel=1e-13)
    assert learn.log1m_tanh2(0.0) == 0.0


def test_squash_density_integrates_to_one():
    """The tanh-squashed Gaussian's log pi (K = 1) is a density on (-1, 1): the integral of
    exp(log pi(a)) da is 1 (scipy quadrature; a = tanh(z + sigma eps) -> eps = (atanh a - z) / sigma),
    which fixes the Gaussian constant and the sign of the log-det term; its mean is E[tanh(z + sigma
    N)] (Gauss-Hermite quadrature); K = 2 log pi is the sum over the two entries."""
    from scipy import integrate
    for z, sigma in ((0.3, 0.5), (-1.2, 0.1), (2.0, 1.0)):
        def dens(a):
            e = (math.atanh(a) - z) / sigma
            return math.exp(learn.squash([[z]], [[e]], sigma)[1][0])
        tot, _ = integrate.quad(dens, -1.0, 1.0, limit=400, points=[math.tanh(z)])
        assert tot == pytest.approx(1.0, abs=1e-7), (z, sigma)
        mean, _ = integrate.quad(lambda a: a * dens(a), -1.0, 1.0, limit=400, points=[math.tanh(z)])
        x, w = np.polynomial.hermite_e.hermegauss(60)
        assert mean == pytest.approx(float(np.sum(w * np.tanh(z + sigma * x)) / math.sqrt(2 * math.pi)), abs=1e-7)
    a2, lp2 = learn.squash([[0.1, -0.4]], [[0.5, 1.5]], 0.2)
    a0, lp0 = learn.squash([[0.1]], [[0.5]], 0.2)
    a1, lp1 = learn.squash([[-0.4]], [[1.5]], 0.2)
    assert lp2[0] == pytest.approx(lp0[0] + lp1[0], rel=1e-14) and a2[0] == [a0[0][0], a1[0][0]]
    a, lp = learn.squash([[0.25, -3.0]])                    # DDPG: a = tanh(z), no density
    assert a[0] == [math.tanh(0.25), math.tanh(-3.0)] and lp is None


def test_dense_forward_and_backward():
    """dense_forward equals its loops; dense_backward_np's parameter and input gradients of
    sum g_out . out against central finite differences of dense_forward (a critic with a scalar
    output and one with 3 outputs)."""
    rng = np.random.default_rng(17)
    for dims in ((6, 7, 5, 1), (4, 5, 6, 3)):
        layers = _tiny_net(rng, dims)
        B = 5
        x = rng.normal(size=(B, dims[0]))
        h1, h2, out = learn.dense_forward(layers, x)
        np.testing.assert_allclose(out, learn.dense_forward_loops(layers, x.tolist()), rtol=1e-13, atol=1e-14)
        g = rng.normal(size=out.shape)
        grads, gx = learn.dense_backward_np(layers, x, h1, h2, g)

        def f():
            return float(np.sum(g * learn.dense_forward(layers, x)[2]))
        h = 1e-6
        for li in range(3):
            for which in (0, 1):
                p = layers[li][which]
                for idx in np.ndindex(p.shape):
                    old = p[idx]
                    p[idx] = old + h
                    fp = f()
                    p[idx] = old - h
                    fm = f()
                    p[idx] = old
                    assert abs((fp - fm) / (2 * h) - grads[li][which][idx]) <= 1e-6 * max(1.0, abs(fp)), (li, which, idx)
        for idx in np.ndindex(x.shape):
            old = x[idx]
            x[idx] = old + h
            fp = f()
            x[idx] = old - h
            fm = f()
            x[idx] = old
            assert abs((fp - fm) / (2 * h) - gx[idx]) <= 1e-6 * max(1.0, abs(fp)), idx


def test_critic_targets_spec_cases():
    """done = 1 -> y = r; alpha = 0 and identical twin critics -> the DDPG-style
    target; Q1' < Q2' everywhere -> the target uses Q1'; a worked SAC value."""
    r, q1, q2, lp = [0.5, -1.0], [2.0, 4.0], [3.0, 1.0], [-0.7, 0.2]
    assert learn.critic_targets(r, [1, 1], q1, 0.99, q2, lp, 0.2) == r
    assert learn.critic_targets(r, [0, 0], q1, 0.9, q1, lp, 0.0) == learn.critic_targets(r, [0, 0], q1, 0.9)
    assert learn.critic_targets([0.0], [0], [1.0], 1.0, [5.0]) == [1.0]
    y = learn.critic_targets(r, [0, 0], q1, 0.9, q2, lp, 0.2)
    assert y == [0.5 + 0.9 * (2.0 + 0.2 * 0.7), -1.0 + 0.9 * (1.0 - 0.2 * 0.2)]
    L, g = learn.critic_head([1.0, 3.0], [0.0, 1.0])
    assert L == 2.5 and g == [1.0, 2.0]


def _critic_q(critic, x, a):
    return learn.dense_forward(critic, np.concatenate([x, a], axis=1))[2][:, 0]


def test_actor_heads_against_finite_differences():
    """The DDPG and SAC actor gradients dL/dz (heads fed with the critics' action gradients from
    dense_backward_np) against central finite differences of the composed float64 losses
    L_mu(z) = -(1/B) sum Q(s, tanh z) and L_pi(z) = (1/B) sum [alpha log pi - min(Q1, Q2)](s,
    tanh(z + sigma eps)); the SAC batch has samples on both sides of the min."""
    rng = np.random.default_rng(23)
    B, S, K = 6, 5, 3
    x = rng.normal(size=(B, S))
    z = rng.normal(0, 0.8, (B, K))
    eps = rng.normal(size=(B, K))
    c1 = _tiny_net(rng, (S + K, 7, 6, 1))
    c2 = _tiny_net(rng, (S + K, 7, 6, 1))
    sigma, alpha = 0.3, 0.2

    def qgrad(critic, a):
        xa = np.concatenate([x, np.asarray(a)], axis=1)
        h1, h2, out = learn.dense_forward(critic, xa)
        _, gx = learn.dense_backward_np(critic, xa, h1, h2, np.ones((B, 1)))
        return out[:, 0], gx[:, S:]

    def l_ddpg(zz):
        a, _ = learn.squash(zz.tolist())
        return -float(np.mean(_critic_q(c1, x, np.array(a))))

    def l_sac(zz):
        a, lp = learn.squash(zz.tolist(), eps.tolist(), sigma)
        q = np.minimum(_critic_q(c1, x, np.array(a)), _critic_q(c2, x, np.array(a)))
        return float(np.mean(alpha * np.array(lp) - q))

    a, _ = learn.squash(z.tolist())
    q, dq = qgrad(c1, a)
    L, g = learn.ddpg_actor_head(a, q, dq)
    assert L == pytest.approx(l_ddpg(z), rel=1e-13)
    a, lp = learn.squash(z.tolist(), eps.tolist(), sigma)
    q1, _ = qgrad(c1, a)
    q2, _ = qgrad(c2, a)
    c2[2][1][0] += float(np.median(q1 - q2))            # shift Q2 so the min switches inside the batch
    q1, d1 = qgrad(c1, a)
    q2, d2 = qgrad(c2, a)
    assert np.any(q1 < q2) and np.any(q2 < q1)
    Ls, gs = learn.sac_actor_head(a, lp, q1, d1, q2, d2, alpha)
    assert Ls == pytest.approx(l_sac(z), rel=1e-13)
    h = 1e-6
    for fn, gg in ((l_ddpg, g), (l_sac, gs)):
        for idx in np.ndindex(z.shape):
            old = z[idx]
            z[idx] = old + h
            fp = fn(z)
            z[idx] = old - h
            fm = fn(z)
            z[idx] = old
            assert abs((fp - fm) / (2 * h) - gg[idx[0]][idx[1]]) <= 1e-7 * max(1.0, abs(fp)), (fn.__name__, idx)


def test_critic_loss_gradient_against_finite_differences():
    """d L_Q / d theta (critic_head's dL/dq through dense_backward_np) against central finite
    differences of the float64 critic loss with the target held fixed."""
    rng = np.random.default_rng(29)
    B, D = 7, 6
    critic = _tiny_net(rng, (D, 5, 4, 1))
    x = rng.normal(size=(B, D))
    y = rng.normal(size=B).tolist()

    def loss():
        return learn.critic_head(learn.dense_forward(critic, x)[2][:, 0].tolist(), y)[0]

    h1, h2, out = learn.dense_forward(critic, x)
    _, g = learn.critic_head(out[:, 0].tolist(), y)
    grads, _ = learn.dense_backward_np(critic, x, h1, h2, np.array(g)[:, None])
    h = 1e-6
    for li in range(3):
        for which in (0, 1):
            p = critic[li][which]
            for idx in np.ndindex(p.shape):
                old = p[idx]
                p[idx] = old + h
                lp = loss()
                p[idx] = old - h
                lm = loss()
                p[idx] = old
                assert abs((lp - lm) / (2 * h) - grads[li][which][idx]) <= 1e-6 * max(1.0, abs(lp)), (li, which, idx)


def test_soft_update_cases():
    """tau = 1 copies the online weights, tau = 0 keeps the target; tau = 0.005 is the float64
    convex combination rounded once."""
    t = np.array([1.0, -2.0, 3.5], dtype=np.float32)
    o = np.array([0.25, 4.0, -1.0], dtype=np.float32)
    assert np.array_equal(learn.soft_update(t, o, 1.0), o)
    assert np.array_equal(learn.soft_update(t, o, 0.0), t)
    assert np.array_equal(learn.soft_update(t, o, 0.005),
                          np.array([0.005 * 0.25 + 0.995 * 1.0, 0.005 * 4.0 + 0.995 * -2.0,
                                    0.005 * -1.0 + 0.995 * 3.5], dtype=np.float32))
