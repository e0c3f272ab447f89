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
