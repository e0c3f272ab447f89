"""Consumer-side oracle pieces (test infrastructure only).

The learner consumes the rollout's T x N x D tensors.
Two of its steps act on those tensors directly, with no backward pass:

* Generalised advantage estimation (the paper names PPO, whose
  standard estimator this is -- reading R-GAE):
      delta_t = r_t + gamma V_{t+1} (1 - d_t) - V_t
      A_t     = delta_t + gamma lambda (1 - d_t) A_{t+1},   A_T = 0
      R_t     = A_t + V_t
  per env, t = T-1 down to 0, V [T+1][N] (V_T = the bootstrap value of the last state);
  optional batch normalisation A' = (A - mean) / std over all T N entries (population
  std; A - mean when std = 0).
* The KL diversity term of Eq. 5: L_new(theta_i) = L(theta_i)
      - lambda sum_{j != i} KL(pi_j || pi_i)
  with the KL of the members' action distributions averaged over a batch of states
  (SPEC S:432-437): diagonal Gaussians with a shared std sigma (PPO, and DDPG wrapped as
  N(mu, sigma)) give KL = sum_k (mu_j,k - mu_i,k)^2 / (2 sigma^2); categorical (DQN
  family, softmax of Q) give sum_a p_j,a (ln p_j,a - ln p_i,a).
Plain float64 loops in the order written.
"""
from __future__ import annotations

import math


def gae(rewards, values, dones, gamma: float, lam: float):
    """rewards / dones [T][N], values [T+1][N] (nested lists or arrays) -> (A, R) [T][N] lists."""
    T = len(rewards)
    N = len(rewards[0]) if T else 0
    A = [[0.0] * N for _ in range(T)]
    R = [[0.0] * N for _ in range(T)]
    for i in range(N):
        nxt = 0.0
        for t in range(T - 1, -1, -1):
            keep = 0.0 if dones[t][i] else 1.0
            delta = float(rewards[t][i]) + gamma * float(values[t + 1][i]) * keep - float(values[t][i])
            nxt = delta + gamma * lam * keep * nxt
            A[t][i] = nxt
            R[t][i] = nxt + float(values[t][i])
    return A, R


def gae_direct(rewards, values, dones, gamma: float, lam: float):
    """O(T^2) direct sum (pin for ``gae``): A_t = sum_{l >= 0} (gamma lambda)^l delta_{t+l},
    truncated at the first done at or after t (the done step's own delta is included)."""
    T = len(rewards)
    N = len(rewards[0]) if T else 0
    A = [[0.0] * N for _ in range(T)]
    for i in range(N):
        for t in range(T):
            s = 0.0
            w = 1.0
            for u in range(t, T):
                keep = 0.0 if dones[u][i] else 1.0
                delta = float(rewards[u][i]) + gamma * float(values[u + 1][i]) * keep - float(values[u][i])
                s += w * delta
                if dones[u][i]:
                    break
                w *= gamma * lam
            A[t][i] = s
    return A


def normalise(A):
    """(A - mean) / std over every entry (population std, two passes); A - mean if std = 0."""
    flat = [a for row in A for a in row]
    n = len(flat)
    m = 0.0
    for a in flat:
        m += a
    m /= n
    q = 0.0
    for a in flat:
        q += (a - m) * (a - m)
    sd = math.sqrt(q / n)
    return [[(a - m) / sd if sd > 0.0 else a - m for a in row] for row in A]


def kl_gaussian(mu_j, mu_i, sigma: float) -> float:
    """KL(N(mu_j, sigma^2 I) || N(mu_i, sigma^2 I)) for one state."""
    s = 0.0
    for a, b in zip(mu_j, mu_i):
        s += (a - b) * (a - b)
    return s / (2.0 * sigma * sigma)


def kl_categorical(q_j, q_i) -> float:
    """KL(softmax(q_j) || softmax(q_i)) for one state."""
    def logsoftmax(q):
        m = max(q)
        z = math.log(sum(math.exp(x - m) for x in q)) + m
        return [x - z for x in q]
    lj, li = logsoftmax(q_j), logsoftmax(q_i)
    return sum(math.exp(a) * (a - b) for a, b in zip(lj, li))


def kl_diversity(outputs, sigma: float, categorical: bool = False):
    """outputs [M][B][K] (per member and state: Gaussian means, or Q-values) ->
    D [M][M] with D[i][j] = mean_s KL(pi_j || pi_i) (the Eq. 5 term of member i is
    lambda sum_{j != i} D[i][j]; D[i][i] = 0)."""
    M = len(outputs)
    B = len(outputs[0])
    D = [[0.0] * M for _ in range(M)]
    for i in range(M):
        for j in range(M):
            if i == j:
                continue
            s = 0.0
            for b in range(B):
                s += (kl_categorical(outputs[j][b], outputs[i][b]) if categorical
                      else kl_gaussian(outputs[j][b], outputs[i][b], sigma))
            D[i][j] = s / B
    return D
