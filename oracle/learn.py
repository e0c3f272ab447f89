"""Consumer-side oracle pieces (test infrastructure only).

The learner consumes the rollout's T x N x D tensors.
Two of its steps act on those tensors directly, with no backward pass (the policy-gradient
step of Eq. 3-4 with the PPO surrogate, its backward pass through the MLP and Adam follow
further down):

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
import numpy as np


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


# ---------------------------------------------------------------- the policy-gradient step
# PAPER.md Eq. 3-4: grad J = E[sum_t R grad log pi(a_t | s_t)], estimated by Monte
# Carlo over the N trajectories of the rollout.  The PPO member replaces R by advantages
# and the likelihood-ratio term by the clipped surrogate (reading R-PPO):
#   log pi(a | s) = sum_k -(a_k - mu_k)^2 / (2 sigma^2) - K ln(sigma sqrt(2 pi)),  mu = tanh(z3(s))
#                   (the Gaussian member of R17: fixed std sigma around the tanh mean, a the
#                   pre-clip continuous action the rollout drew)
#   rho = exp(log pi_new - log pi_old)
#   L   = (1/B) sum_s min(rho_s A_s, clip(rho_s, 1 - eps, 1 + eps) A_s)        (maximised)
#   dL/dtheta = (1/B) sum_s c_s grad log pi(a_s | s_s),  c_s = rho_s A_s when the unclipped term
#               is the minimum (not (A > 0 and rho > 1 + eps), not (A < 0 and rho < 1 - eps)),
#               else 0;  d log pi / d z3 = ((a - mu) / sigma^2) (1 - mu^2)
# The loss the optimiser minimises is -L; its gradient flows back through the MLP of oracle.mlp
# (ReLU hidden layers) with the hidden activations given (straight-through for the bf16 rounding
# the rollout applies: the same activations the device forward produced).

def ppo_head(z3, a, logp_old, adv, sigma: float = 0.1, eps: float = 0.2):
    """Per sample s (rows of z3 / a [B][K], logp_old / adv [B]): returns
    (logp_new [B], rho [B], coef [B], g3 [B][K] = d(-L)/dz3, L) in float64 with plain loops."""
    B, K = len(z3), len(z3[0])
    const = K * math.log(sigma * math.sqrt(2.0 * math.pi))
    logp, rho, coef = [0.0] * B, [0.0] * B, [0.0] * B
    g3 = [[0.0] * K for _ in range(B)]
    L = 0.0
    for s in range(B):
        mu = [math.tanh(float(z3[s][k])) for k in range(K)]
        q = 0.0
        for k in range(K):
            d = float(a[s][k]) - mu[k]
            q += d * d
        logp[s] = -q / (2.0 * sigma * sigma) - const
        rho[s] = math.exp(logp[s] - float(logp_old[s]))
        A = float(adv[s])
        clipped = min(max(rho[s], 1.0 - eps), 1.0 + eps)
        L += min(rho[s] * A, clipped * A)
        active = not ((A > 0.0 and rho[s] > 1.0 + eps) or (A < 0.0 and rho[s] < 1.0 - eps))
        coef[s] = rho[s] * A if active else 0.0
        for k in range(K):
            g3[s][k] = -coef[s] / B * ((float(a[s][k]) - mu[k]) / (sigma * sigma)) * (1.0 - mu[k] * mu[k])
    return logp, rho, coef, g3, L / B


def mlp_backward(layers64, x, hidden, g_out):
    """Gradients of sum_s g_out[s] . z_out(s) for the 3-layer ReLU MLP of oracle.mlp, given the
    input x [B][in], the hidden activations hidden [B][2][H] (the values each next layer consumed)
    and g_out [B][out] = d loss / d z_out.  Returns [(dW_l [out][in], db_l [out]) for l = 1..3],
    float64, plain loops over samples and units (small B only; ``mlp_backward_np`` is the
    vectorised restatement pinned against it)."""
    (w1, _), (w2, _), (w3, _) = layers64
    H1, H2, O = w1.shape[0], w2.shape[0], w3.shape[0]
    B = len(x)
    dW = [np.zeros_like(w1), np.zeros_like(w2), np.zeros_like(w3)]
    db = [np.zeros(H1), np.zeros(H2), np.zeros(O)]
    for s in range(B):
        h1 = [float(v) for v in hidden[s][0][:H1]]
        h2 = [float(v) for v in hidden[s][1][:H2]]
        g3 = [float(v) for v in g_out[s]]
        g2 = [0.0] * H2
        for j in range(H2):
            if h2[j] > 0.0:
                acc = 0.0
                for o in range(O):
                    acc += g3[o] * w3[o, j]
                g2[j] = acc
        g1 = [0.0] * H1
        for i in range(H1):
            if h1[i] > 0.0:
                acc = 0.0
                for j in range(H2):
                    acc += g2[j] * w2[j, i]
                g1[i] = acc
        for o in range(O):
            db[2][o] += g3[o]
            for j in range(H2):
                dW[2][o, j] += g3[o] * h2[j]
        for j in range(H2):
            db[1][j] += g2[j]
            for i in range(H1):
                dW[1][j, i] += g2[j] * h1[i]
        xs = [float(v) for v in x[s]]
        for i in range(H1):
            db[0][i] += g1[i]
            for c in range(w1.shape[1]):
                dW[0][i, c] += g1[i] * xs[c]
    return [(dW[l], db[l]) for l in range(3)]


def mlp_backward_np(layers64, x, hidden, g_out):
    """The same gradients with NumPy matrix products (library primitive ``@``)."""
    (w1, _), (w2, _), (w3, _) = layers64
    H1, H2 = w1.shape[0], w2.shape[0]
    x = np.asarray(x, dtype=np.float64)
    h1 = np.asarray(hidden, dtype=np.float64)[:, 0, :H1]
    h2 = np.asarray(hidden, dtype=np.float64)[:, 1, :H2]
    g3 = np.asarray(g_out, dtype=np.float64)
    g2 = (g3 @ w3) * (h2 > 0)
    g1 = (g2 @ w2) * (h1 > 0)
    return [(g1.T @ x, g1.sum(0)), (g2.T @ h1, g2.sum(0)), (g3.T @ h2, g3.sum(0))]


def adam(theta, m, v, g, step: int, lr: float = 3e-4, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8):
    """One Adam step (Kingma & Ba) on flat float64 lists, ``step`` >= 1 the 1-based count:
    m <- b1 m + (1 - b1) g; v <- b2 v + (1 - b2) g^2; theta <- theta - lr mhat / (sqrt(vhat) + eps)
    with mhat = m / (1 - b1^step), vhat = v / (1 - b2^step).  Returns new (theta, m, v)."""
    c1 = 1.0 - beta1 ** step
    c2 = 1.0 - beta2 ** step
    th, mm, vv = list(theta), list(m), list(v)
    for i in range(len(th)):
        mm[i] = beta1 * mm[i] + (1.0 - beta1) * g[i]
        vv[i] = beta2 * vv[i] + (1.0 - beta2) * g[i] * g[i]
        th[i] = th[i] - lr * (mm[i] / c1) / (math.sqrt(vv[i] / c2) + eps)
    return th, mm, vv


# ---------------------------------------------------------------- the DQN family's update (R-DQN)
# PAPER.md P:317-321, P:346 (DQN, Double DQN, Dueling DQN members of the crypto ensemble); SPEC
# S:362-391.  For a batch of transitions (s, a, r, done, s'):
#   DQN:        y = r + gamma (1 - done) max_a' Q_target(s', a')
#   Double DQN: y = r + gamma (1 - done) Q_target(s', argmax_a' Q_online(s', a'))   (lowest index on ties)
#   Dueling:    the network's outputs are (A_0, A_1, A_2, V) and Q(s, a) = V + A_a - mean_j A_j
#   loss:       L = (1/B) sum_s (Q(s, a_s) - y_s)^2  (y is a constant: no gradient through the target)
#   dL/d out:   plain nets: 2 (Q - y) / B on output a_s;  dueling: 2 (Q - y) / B (delta_{a j} - 1/3) on
#               A_j and 2 (Q - y) / B on V
# then the same backward pass through the MLP (mlp_backward) and Adam.

def dueling_q(out):
    """out [A_0 .. A_{n-1}, V] -> Q [n] = V + A - mean A."""
    n = len(out) - 1
    m = 0.0
    for j in range(n):
        m += out[j]
    m /= n
    return [out[n] + out[j] - m for j in range(n)]


def q_values(out, dueling: bool):
    return dueling_q(out) if dueling else list(out)


def dqn_targets(q_next_target, r, done, gamma: float, q_next_online=None, dueling: bool = False):
    """y [B] from the target net's outputs at s' (and the online net's for Double DQN)."""
    y = []
    for s in range(len(r)):
        qt = q_values([float(v) for v in q_next_target[s]], dueling)
        if q_next_online is None:
            boot = max(qt)
        else:
            qo = q_values([float(v) for v in q_next_online[s]], dueling)
            best = 0
            for j in range(1, len(qo)):
                if qo[j] > qo[best]:
                    best = j
            boot = qt[best]
        keep = 0.0 if done[s] else 1.0
        y.append(float(r[s]) + gamma * keep * boot)
    return y


def dqn_head(out, a, y, dueling: bool = False):
    """(L, g_out [B][O]) for the online net's outputs ``out`` at s and actions a [B]."""
    B, O = len(out), len(out[0])
    g = [[0.0] * O for _ in range(B)]
    L = 0.0
    for s in range(B):
        q = q_values([float(v) for v in out[s]], dueling)
        d = q[int(a[s])] - float(y[s])
        L += d * d
        c = 2.0 * d / B
        if dueling:
            n = O - 1
            for j in range(n):
                g[s][j] = c * ((1.0 if j == int(a[s]) else 0.0) - 1.0 / n)
            g[s][n] = c
        else:
            g[s][int(a[s])] = c
    return L / B, g


# ---------------------------------------------------------------- the actor-critic updates (R-AC)
# The stock ensemble's DDPG and SAC members (reading
# R-AC).  A critic Q(s, a) is a 3-layer ReLU MLP on the concatenated input [x(s); a] with a linear
# scalar output (a learner-only network: float32 weights, no bf16 quantisation; ``dense_forward``).
# The actor is the rollout's policy MLP z(s) (oracle.mlp), its action head that of R17:
#   DDPG: a = mu(s) = tanh(z(s))
#         y    = r + gamma (1 - done) Q_targ(s', tanh(z_targ(s')))
#         L_Q  = (1/B) sum_s (Q(s, a_s) - y_s)^2                         (y held fixed)
#         L_mu = -(1/B) sum_s Q(s, tanh(z(s)));   dL_mu/dz_k = -(1/B) dQ/da_k (1 - a_k^2)
#   SAC (fixed std sigma around the pre-tanh mean, R17; fixed temperature alpha):
#         u = z(s) + sigma eps,  a = tanh(u)
#         log pi(a|s) = sum_k [-eps_k^2 / 2 - ln(sigma sqrt(2 pi)) - ln(1 - tanh(u_k)^2)]
#                       with ln(1 - tanh(u)^2) = 2 (ln 2 - u - softplus(-2 u))  (the stable form)
#         y    = r + gamma (1 - done) (min(Q1_targ, Q2_targ)(s', a') - alpha log pi(a'|s')),
#                a' = tanh(z(s') + sigma eps') a fresh sample
#         L_Qi = (1/B) sum_s (Qi(s, a_s) - y_s)^2,  i = 1, 2
#         L_pi = (1/B) sum_s [alpha log pi(a~|s) - min(Q1, Q2)(s, a~)],  a~ = tanh(z(s) + sigma eps)
#         dL_pi/dz_k = (1/B) [2 alpha a~_k - dQm/da_k (1 - a~_k^2)],  Qm the smaller critic at
#                      (s, a~) (Q1 on ties); at fixed eps the Gaussian term of log pi does not move
#                      with z, and d/du [-ln(1 - tanh(u)^2)] = 2 tanh(u)
#   Soft target update: theta_targ <- tau theta + (1 - tau) theta_targ (tau = 0.005), float64,
#   one rounding to float32.

def softplus(x: float) -> float:
    """ln(1 + e^x) without overflow."""
    return max(x, 0.0) + math.log1p(math.exp(-abs(x)))


def log1m_tanh2(u: float) -> float:
    """ln(1 - tanh(u)^2) = 2 (ln 2 - u - softplus(-2 u)) (finite for every finite u)."""
    return 2.0 * (math.log(2.0) - u - softplus(-2.0 * u))


def squash(z, eps=None, sigma: float = 0.1):
    """Rows z [B][K]: a = tanh(z + sigma eps) and log pi(a|s) [B] (SAC), or a = tanh(z) and no
    log-density (DDPG, eps None).  float64 loops."""
    B, K = len(z), len(z[0])
    a = [[0.0] * K for _ in range(B)]
    logp = None if eps is None else [0.0] * B
    c = math.log(sigma * math.sqrt(2.0 * math.pi))
    for s in range(B):
        acc = 0.0
        for k in range(K):
            e = 0.0 if eps is None else float(eps[s][k])
            u = float(z[s][k]) + sigma * e
            a[s][k] = math.tanh(u)
            if eps is not None:
                acc += -0.5 * e * e - c - log1m_tanh2(u)
        if eps is not None:
            logp[s] = acc
    return a, logp


def dense_forward(layers64, x):
    """Critic forward, float64 with no quantisation: [(W [out][in], b [out])] x 3, x [B][in] ->
    (h1 [B][H1], h2 [B][H2], out [B][O]); h = ReLU(W x + b) for the hidden layers, the last
    linear.  The matrix product is the library primitive ``@`` (pinned against the loops)."""
    (w1, b1), (w2, b2), (w3, b3) = layers64
    x = np.asarray(x, dtype=np.float64)
    h1 = np.maximum(x @ w1.T + b1, 0.0)
    h2 = np.maximum(h1 @ w2.T + b2, 0.0)
    return h1, h2, h2 @ w3.T + b3


def dense_forward_loops(layers64, x):
    """``dense_forward`` with explicit loops (small cases)."""
    out = []
    for row in x:
        h = [float(v) for v in row]
        for li, (w, b) in enumerate(layers64):
            nxt = []
            for j in range(w.shape[0]):
                acc = float(b[j])
                for i in range(w.shape[1]):
                    acc += float(w[j, i]) * h[i]
                nxt.append(max(acc, 0.0) if li < 2 else acc)
            h = nxt
        out.append(h)
    return np.array(out)


def dense_backward_np(layers64, x, h1, h2, g_out):
    """Gradients of sum_s g_out[s] . out(s) of ``dense_forward``: ([(dW_l, db_l)] for l = 1..3,
    g_x [B][in]); ReLU derivative 1 where the activation is > 0."""
    (w1, _), (w2, _), (w3, _) = layers64
    x = np.asarray(x, dtype=np.float64)
    g3 = np.asarray(g_out, dtype=np.float64)
    g2 = (g3 @ w3) * (h2 > 0)
    g1 = (g2 @ w2) * (h1 > 0)
    return [(g1.T @ x, g1.sum(0)), (g2.T @ h1, g2.sum(0)), (g3.T @ h2, g3.sum(0))], g1 @ w1


def critic_targets(r, done, q1_next, gamma: float, q2_next=None, logp_next=None, alpha: float = 0.0):
    """y [B] = r + gamma (1 - done) (min(q1', q2') - alpha log pi'), q2' / log pi' optional (DDPG:
    y = r + gamma (1 - done) q')."""
    y = []
    for s in range(len(r)):
        boot = float(q1_next[s])
        if q2_next is not None and float(q2_next[s]) < boot:
            boot = float(q2_next[s])
        if logp_next is not None:
            boot = boot - alpha * float(logp_next[s])
        keep = 0.0 if done[s] else 1.0
        y.append(float(r[s]) + gamma * keep * boot)
    return y


def critic_head(q, y):
    """(L = (1/B) sum (q - y)^2, g [B] = dL/dq = 2 (q - y) / B)."""
    B = len(q)
    L = 0.0
    g = [0.0] * B
    for s in range(B):
        d = float(q[s]) - float(y[s])
        L += d * d
        g[s] = 2.0 * d / B
    return L / B, g


def ddpg_actor_head(a, q, dq):
    """(L_mu = -(1/B) sum q, g_z [B][K] = -(1/B) dq (1 - a^2)) for a = tanh(z), the critic's value q
    [B] and its gradient dq [B][K] = dQ/da at (s, a)."""
    B, K = len(a), len(a[0])
    L = 0.0
    g = [[0.0] * K for _ in range(B)]
    for s in range(B):
        L -= float(q[s])
        for k in range(K):
            g[s][k] = -float(dq[s][k]) * (1.0 - a[s][k] * a[s][k]) / B
    return L / B, g


def sac_actor_head(a, logp, q1, dq1, q2, dq2, alpha: float):
    """(L_pi, g_z [B][K]) of R-AC for the reparameterised sample a = tanh(z + sigma eps), its log pi,
    and both critics' values / action gradients at (s, a)."""
    B, K = len(a), len(a[0])
    L = 0.0
    g = [[0.0] * K for _ in range(B)]
    for s in range(B):
        two = q2 is not None and float(q2[s]) < float(q1[s])
        qm = float(q2[s]) if two else float(q1[s])
        dqm = dq2[s] if two else dq1[s]
        L += alpha * float(logp[s]) - qm
        for k in range(K):
            g[s][k] = (2.0 * alpha * a[s][k] - float(dqm[k]) * (1.0 - a[s][k] * a[s][k])) / B
    return L / B, g


def soft_update(target, online, tau: float):
    """float32 target <- f32(tau theta + (1 - tau) theta_target), the sum in float64."""
    t = np.asarray(target, dtype=np.float64)
    o = np.asarray(online, dtype=np.float64)
    return (tau * o + (1.0 - tau) * t).astype(np.float32)
