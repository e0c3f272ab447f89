"""Pins for the ensemble rules of oracle/policy.py -- CPU only.

softmax_weights: PAPER.md §5.2.1 P:309 ("agents with very low Sharpe ratios are discarded;
weights ... a softmax function applied to their Sharpe ratios"), examples SPEC S:499-501.
majority_vote: §5.2.2, examples SPEC S:519-521.  dueling_q: Wang et al.'s head.
condorcet_probability: Eq. 1, examples SPEC S:529-531.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import policy


# ------------------------------------------------------------------ softmax weights
def test_softmax_weights_spec_examples():
    assert policy.softmax_weights([0.3, 0.3, 0.3]) == pytest.approx([1 / 3] * 3, abs=1e-15)
    w = policy.softmax_weights([1.0, 0.0], threshold=-math.inf, temperature=1.0)
    e = math.e
    assert w == pytest.approx([e / (e + 1), 1 / (e + 1)], abs=1e-15)      # 0.731 / 0.269
    assert policy.softmax_weights([0.5, -0.2], threshold=0.0) == [1.0, 0.0]


def test_softmax_weights_closed_form_and_gating():
    rng = np.random.default_rng(3)
    for _ in range(200):
        m = int(rng.integers(1, 31))
        s = list(rng.normal(0.2, 1.0, m))
        thr = float(rng.normal(0.0, 0.5))
        tau = float(rng.uniform(0.2, 3.0))
        w = policy.softmax_weights(s, thr, tau)
        keep = [x >= thr for x in s]
        if any(keep):
            # direct definition exp(s_i / tau) / sum over kept (no max shift), in Fractions of floats
            den = sum(math.exp(x / tau) for x, k in zip(s, keep) if k)
            ref = [math.exp(x / tau) / den if k else 0.0 for x, k in zip(s, keep)]
            assert w == pytest.approx(ref, rel=1e-12, abs=1e-300)
        else:
            best = int(np.argmax(s))
            assert w == [1.0 if i == best else 0.0 for i in range(m)]
        assert sum(w) == pytest.approx(1.0, abs=1e-12)                       # simplex
        assert all(x >= 0 for x in w)


def test_softmax_weights_monotone_and_scale_invariant():
    s = [0.4, 1.1, 0.7, -0.3]
    w0 = policy.softmax_weights(s, threshold=-1.0)
    w1 = policy.softmax_weights([0.4, 1.1, 0.9, -0.3], threshold=-1.0)     # raise member 2
    assert w1[2] > w0[2]
    w2 = policy.softmax_weights([3 * x for x in s], threshold=-3.0, temperature=3.0)
    assert w2 == pytest.approx(w0, rel=1e-12)
    # NaN Sharpes (std = 0, reading R21) are discarded
    assert policy.softmax_weights([float("nan"), 0.2]) == [0.0, 1.0]


# ------------------------------------------------------------------ majority vote
def test_majority_vote_spec_examples():
    assert policy.majority_vote([1, 1, -1]) == 1                  # {buy, buy, sell} -> buy
    assert policy.majority_vote([1, -1]) == -1                    # tie, no hold: lower index (sell)
    assert policy.majority_vote([1, 0]) == 0                      # tie with hold: hold
    assert policy.majority_vote([0, 0, 0]) == 0 and policy.majority_vote([-1]) == -1


def test_majority_vote_brute_force_and_permutation_invariance():
    for m in range(1, 7):
        for votes in itertools.product((-1, 0, 1), repeat=m):
            r = policy.majority_vote(list(votes))
            c = {v: votes.count(v) for v in (-1, 0, 1)}
            top = max(c.values())
            assert c[r] == top                                          # a plurality winner
            if c[0] == top:
                assert r == 0                                           # hold wins its ties
            elif c[-1] == top:
                assert r == -1                                          # then the lower index
            for perm in set(itertools.permutations(votes)):
                assert policy.majority_vote(list(perm)) == r


# ------------------------------------------------------------------ dueling head
def test_dueling_head_identities():
    rng = np.random.default_rng(5)
    for _ in range(500):
        a = list(rng.normal(0, 1, 3))
        v = float(rng.normal(0, 1))
        q = policy.dueling_q(a, v)
        assert sum(q) / 3 == pytest.approx(v, abs=1e-12)                # mean_j Q_j = V
        assert policy.argmax_lowest(q) == policy.argmax_lowest(a)        # greedy action from A
    assert policy.dueling_q([0.0, 0.0, 0.0], 2.5) == [2.5, 2.5, 2.5]


# ------------------------------------------------------------------ Condorcet (Eq. 1)
def test_condorcet_probability():
    assert policy.condorcet_probability(1, 0.37) == pytest.approx(0.37, abs=1e-15)
    assert policy.condorcet_probability(3, 0.6) == pytest.approx(0.648, abs=1e-12)
    for n in (1, 3, 5, 21, 101):
        assert policy.condorcet_probability(n, 0.5) == pytest.approx(0.5, abs=1e-12)
    # exact rational tail for n = 7, p = 3/5
    p = Fraction(3, 5)
    exact = sum(math.comb(7, k) * p ** k * (1 - p) ** (7 - k) for k in range(4, 8))
    assert policy.condorcet_probability(7, 0.6) == pytest.approx(float(exact), abs=1e-12)
    prev = 0.0
    for n in range(1, 60, 2):
        cur = policy.condorcet_probability(n, 0.6)
        assert cur > prev
        prev = cur
    assert policy.condorcet_probability(101, 0.6) > 0.97
    with pytest.raises(ValueError):
        policy.condorcet_probability(4, 0.6)
