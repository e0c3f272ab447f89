"""Action sampling and ensemble oracle (test infrastructure only).

* Gaussian policy, C1 and the C2 PPO member (BASELINE.json configs[1]: "tanh output
  scaled to +-100 shares, Gaussian sampling with std 0.1"; readings R17/R18):
      mu = tanh(z);  a = clip(mu + 0.1 eps, -1, 1);  shares = rha(100 a)
* C2 members (configs[2]; readings R17, R19, R20):
      PPO   a_P = clip(tanh(z_P) + 0.1 eps_P, -1, 1)
      SAC   a_S = tanh(z_S + 0.1 eps_S)                       (squashed Gaussian)
      DDPG  x <- x + 0.15 (0 - x) + 0.2 eps_D  (OU, dt=1, update-then-use)
            a_D = clip(tanh(z_D) + x, -1, 1)
      mean  abar = ((a_P + a_S) + a_D) / 3;  shares = rha(100 abar)
  PAPER.md P:300, P:310 ("weighted averaging"; BASELINE binds uniform weights).
* Q argmax (configs[3]): lowest index on ties; epsilon-greedy
  with a supplied uniform pair (u_explore, u_action).
"""
from __future__ import annotations

import math

from .quant import rha

SIGMA = 0.1
OU_THETA = 0.15
OU_SIGMA = 0.2


def clip(x: float, lo: float = -1.0, hi: float = 1.0) -> float:
    return lo if x < lo else hi if x > hi else x


def gaussian_action(z: float, eps: float, std: float = SIGMA) -> float:
    return clip(math.tanh(z) + std * eps)


def sac_action(z: float, eps: float, std: float = SIGMA) -> float:
    return math.tanh(z + std * eps)


def ou_update(x: float, eps: float, theta: float = OU_THETA, sigma: float = OU_SIGMA) -> float:
    return (x + theta * (0.0 - x)) + sigma * eps


def ddpg_action(z: float, x: float) -> float:
    return clip(math.tanh(z) + x)


def shares(a: float, max_trade: int = 100) -> int:
    return rha(max_trade * a)


def ensemble_mean(actions) -> float:
    """Uniform mean, summed in member order then divided by M (reading R20)."""
    s = 0.0
    for a in actions:
        s = s + a
    return s / len(actions)


def weighted_mean(actions, weights) -> float:
    s = 0.0
    for a, w in zip(actions, weights):
        s = s + w * a
    return s


def argmax_lowest(q) -> int:
    best = 0
    for j in range(1, len(q)):
        if q[j] > q[best]:
            best = j
    return best


def epsilon_greedy(q, eps: float, u_explore: float, u_action: float) -> int:
    """With probability eps take a uniformly random action, else argmax."""
    n = len(q)
    if u_explore < eps:
        return min(int(u_action * n), n - 1)
    return argmax_lowest(q)


# ------------------------------------------------------------------ SURVEY §8(f) NEXT-1 / NEXT-2
# Stock ensemble weights (§5.2.1): members are validated on a 5-day
# window, "agents with very low Sharpe ratios are discarded", the rest weighted by "a
# softmax function applied to their Sharpe ratios" (Eq. 6 P:305-307 for the ratio).
# Readings (DESIGN.md R-GATE, after SPEC S:496): discard Sharpe < threshold (default
# 0.0; a NaN Sharpe is discarded); softmax at temperature tau over the retained ones;
# if all are discarded, the best finite Sharpe keeps weight 1 (member 0 if none is
# finite).
def softmax_weights(sharpes, threshold: float = 0.0, temperature: float = 1.0):
    keep = [s == s and s >= threshold for s in sharpes]
    if not any(keep):
        finite = [i for i, s in enumerate(sharpes) if s == s]
        best = max(finite, key=lambda i: (sharpes[i], -i)) if finite else 0
        return [1.0 if i == best else 0.0 for i in range(len(sharpes))]
    top = max(s for s, k in zip(sharpes, keep) if k)
    e = [math.exp((s - top) / temperature) if k else 0.0 for s, k in zip(sharpes, keep)]
    tot = 0.0
    for x in e:
        tot = tot + x
    return [x / tot for x in e]


# Crypto ensemble (§5.2.2): "the majority action is selected as the
# final ensemble action".  Plurality over the members' actions; ties go to the action
# closest to 0 (hold), then to the lowest index (reading R-VOTE).
def majority_vote(actions, values=(-1, 0, 1)) -> int:
    counts = {v: 0 for v in values}
    for a in actions:
        counts[a] += 1
    top = max(counts.values())
    tied = [v for v in values if counts[v] == top]
    return min(tied, key=lambda v: (abs(v), values.index(v)))


# Dueling DQN head (Wang et al. 2016, the paper's third crypto member): Q_j = V + A_j -
# mean_j A_j.  Its greedy action is argmax_j A_j (V and the mean do not depend on j).
def dueling_q(a_head, v: float):
    m = 0.0
    for x in a_head:
        m = m + x
    m = m / len(a_head)
    return [v + (x - m) for x in a_head]


# Condorcet's jury theorem, Eq. 1: P(majority of n independent
# voters, each right with probability p, is right) = sum_{k > n/2} C(n,k) p^k (1-p)^(n-k).
def condorcet_probability(n: int, p: float) -> float:
    if n < 1 or n % 2 == 0:
        raise ValueError("n must be a positive odd integer")
    tot = 0.0
    for k in range(n // 2 + 1, n + 1):
        tot = tot + math.comb(n, k) * p ** k * (1.0 - p) ** (n - k)
    return tot
