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
