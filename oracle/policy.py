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
