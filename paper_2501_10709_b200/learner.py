"""The learner's update steps for the DDPG and SAC members over the C ABI (
PAPER.md P:139-146 (the learning phase consumes the rollout's experience), P:78 / P:300 / P:343 (the
PPO, SAC and DDPG members of the stock ensemble); reading R-AC, every formula in
oracle/learn.py).

Argument marshalling and sequencing only: each forward, head, backward, Adam step and soft update
is one library call (libfinenv.so).  A batch is a dict of device tensors: ``x`` / ``x_next`` bf16
bits [B][S] (the observations the rollout fed its policy; fin_gather_observations), ``a`` f32 [B][K]
(the executed continuous action before the share rounding), ``reward`` f32 [B], ``done`` u8 [B];
SAC also takes ``eps`` / ``eps_next`` f32 [B][K] (the reparameterisation noise of a~ and a').

Networks: the actor is a fin policy handle (the rollout's bf16 tcgen05 forward) with float32
master weights and Adam state (``Actor``); critics Q(s, a) are float32 ``DenseNet`` s on the
concatenated input [x; a] (fin_dense_forward / fin_dense_backward).  Targets are copies updated
by fin_soft_update (the actor's target is re-installed with fin_policy_load after its update).
"""
from __future__ import annotations

import math

import numpy as np

from . import fin


def _adam_state(params):
    import torch
    return [(torch.zeros_like(p), torch.zeros_like(p)) for p in params]


class DenseNet:
    """A float32 3-layer ReLU MLP on the device (a critic), its gradient buffers and Adam state."""

    def __init__(self, dims, seed: int, device="cuda"):
        import torch
        rng = np.random.default_rng(seed)
        self.dims = tuple(int(d) for d in dims)
        self.layers = []
        for i, o in zip(self.dims[:-1], self.dims[1:]):
            w = rng.normal(0.0, math.sqrt(2.0 / i), (o, i)).astype(np.float32)
            b = rng.normal(0.0, 0.01, o).astype(np.float32)
            self.layers.append((torch.from_numpy(w).to(device), torch.from_numpy(b).to(device)))
        self.grads = [(torch.zeros_like(w), torch.zeros_like(b)) for w, b in self.layers]
        self.opt = _adam_state(self.params())
        self.step = 0

    def params(self):
        return [t for pair in self.layers for t in pair]

    def grad_list(self):
        return [t for pair in self.grads for t in pair]

    def weights(self):
        return [w for w, _ in self.layers]

    def copy(self, seed: int = 0) -> "DenseNet":
        c = DenseNet(self.dims, seed)
        for (cw, cb), (w, b) in zip(c.layers, self.layers):
            cw.copy_(w)
            cb.copy_(b)
        return c

    def forward(self, x, out, hidden=None, stream=None):
        fin.fin_dense_forward(x, self.layers, out, hidden, stream=stream)

    def adam(self, lr: float, stream=None):
        self.step += 1
        for p, g, (m, v) in zip(self.params(), self.grad_list(), self.opt):
            fin.fin_adam_step(p, m, v, g, self.step, lr=lr, stream=stream)

    def soft_update_from(self, online: "DenseNet", tau: float, stream=None):
        for t, o in zip(self.params(), online.params()):
            fin.fin_soft_update(t, o, tau, stream=stream)


class Actor:
    """A policy handle (bf16 image for the rollout / forward) with float32 master weights."""

    def __init__(self, kind: int, layers_bf16, layers_f32=None):
        import torch
        self.handle = fin.fin_policy_create(kind, layers_bf16)
        self.dims = tuple(self.handle.dims)
        if layers_f32 is None:   # the bf16 values, widened
            layers_f32 = []
            for w, b in layers_bf16:
                wf = (np.asarray(w, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)
                layers_f32.append((wf, np.asarray(b, dtype=np.float32)))
        self.w = [torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32)).cuda() for w, _ in layers_f32]
        self.b = [torch.from_numpy(np.ascontiguousarray(b, dtype=np.float32)).cuda() for _, b in layers_f32]
        self.grads = [(torch.zeros_like(w), torch.zeros_like(b)) for w, b in zip(self.w, self.b)]
        self.opt = _adam_state(self.params())
        self.step = 0
        self.kind = kind

    def params(self):
        return self.w + self.b

    def grad_list(self):
        return [g for g, _ in self.grads] + [g for _, g in self.grads]

    def forward(self, x, z, hidden=None, stream=None):
        fin.fin_mlp_forward(self.handle, x, z, hidden, stream=stream)

    def adam(self, lr: float, stream=None):
        self.step += 1
        for p, g, (m, v) in zip(self.params(), self.grad_list(), self.opt):
            fin.fin_adam_step(p, m, v, g, self.step, lr=lr, stream=stream)

    def load(self, stream=None):
        fin.fin_policy_load(self.handle, self.w, self.b, stream=stream)

    def soft_update_from(self, online: "Actor", tau: float, stream=None):
        for t, o in zip(self.params(), online.params()):
            fin.fin_soft_update(t, o, tau, stream=stream)
        self.load(stream=stream)


def _zeros(shape, dtype):
    import torch
    return torch.zeros(shape, dtype=dtype, device="cuda")


def _q_and_dq(critic: DenseNet, x, a, S: int, stream):
    """Q(s, a) [B] and dQ/d[x; a] [B][S + K] (its last K columns are dQ/da)."""
    import torch
    B, K = int(a.shape[0]), int(a.shape[1])
    xa = _zeros((B, S + K), torch.float32)
    fin.fin_concat_obs_action(x, a, xa, stream=stream)
    hid = _zeros((B, critic.dims[1] + critic.dims[2]), torch.float32)
    q = _zeros((B, 1), torch.float32)
    critic.forward(xa, q, hid, stream=stream)
    gx = _zeros((B, S + K), torch.float32)
    fin.fin_dense_backward(xa, hid, torch.ones((B, 1), dtype=torch.float32, device="cuda"), critic.weights(), g_x=gx,
                           stream=stream)
    return q.view(-1), gx


def _critic_step(critic: DenseNet, x, a, S, batch, q1n, q2n, lpn, gamma, alpha, lr, stream):
    import torch
    B, K = int(a.shape[0]), int(a.shape[1])
    xa = _zeros((B, S + K), torch.float32)
    fin.fin_concat_obs_action(x, a, xa, stream=stream)
    hid = _zeros((B, critic.dims[1] + critic.dims[2]), torch.float32)
    q = _zeros((B, 1), torch.float32)
    critic.forward(xa, q, hid, stream=stream)
    g = _zeros(B, torch.float32)
    st = _zeros(4, torch.float64)
    fin.fin_critic_head(q.view(-1), batch["reward"], batch["done"], q1n, g, st, q2_next=q2n, logp_next=lpn,
                        gamma=gamma, alpha=alpha, stream=stream)
    fin.fin_dense_backward(xa, hid, g.view(B, 1), critic.weights(), grads=critic.grads, stream=stream)
    critic.adam(lr, stream=stream)
    return st


def ddpg_update(actor: Actor, actor_targ: Actor, critic: DenseNet, critic_targ: DenseNet, batch, gamma: float = 0.99,
                tau: float = 0.005, lr_actor: float = 3e-4, lr_critic: float = 3e-4, stream=None):
    """One DDPG update (R-AC): critic regression to y = r + gamma (1 - done) Q_targ(s', tanh z_targ(s')),
    actor ascent on Q(s, tanh z(s)) through the updated critic, soft target updates.  Returns the
    device stats (critic [4], actor [4])."""
    import torch
    x, xn, a = batch["x"], batch["x_next"], batch["a"]
    B, S, K = int(x.shape[0]), int(x.shape[1]), int(a.shape[1])
    H = max(actor.dims[1], actor.dims[2])
    # target: a' = tanh(z_targ(s')), q' = Q_targ(s', a')
    zn = _zeros((B, K), torch.float32)
    actor_targ.forward(xn, zn, stream=stream)
    an = _zeros((B, K), torch.float32)
    fin.fin_squash(zn, an, stream=stream)
    xan = _zeros((B, S + K), torch.float32)
    fin.fin_concat_obs_action(xn, an, xan, stream=stream)
    qn = _zeros((B, 1), torch.float32)
    critic_targ.forward(xan, qn, stream=stream)
    st_c = _critic_step(critic, x, a, S, batch, qn.view(-1), None, None, gamma, 0.0, lr_critic, stream)
    # actor: mu(s) = tanh(z(s)), g_z = -(1/B) dQ/da (1 - mu^2)
    z = _zeros((B, K), torch.float32)
    hid = _zeros((B, 2, H), torch.int16)
    actor.forward(x, z, hid, stream=stream)
    mu = _zeros((B, K), torch.float32)
    fin.fin_squash(z, mu, stream=stream)
    q, gx = _q_and_dq(critic, x, mu, S, stream)
    gz = _zeros((B, K), torch.float32)
    st_a = _zeros(4, torch.float64)
    fin.fin_actor_head(mu, q, gx[:, S:], gz, st_a, stream=stream)
    fin.fin_policy_backward(x, hid, gz, actor.w[1], actor.w[2], actor.grads, stream=stream)
    actor.adam(lr_actor, stream=stream)
    actor.load(stream=stream)
    critic_targ.soft_update_from(critic, tau, stream=stream)
    actor_targ.soft_update_from(actor, tau, stream=stream)
    return st_c, st_a


def sac_update(actor: Actor, critics, critics_targ, batch, sigma: float = 0.1, alpha: float = 0.2,
               gamma: float = 0.99, tau: float = 0.005, lr_actor: float = 3e-4, lr_critic: float = 3e-4, stream=None):
    """One SAC update (R-AC) with twin critics: y = r + gamma (1 - done) (min Q_targ(s', a') - alpha
    log pi(a'|s')), a' = tanh(z(s') + sigma eps'); each critic regresses to y; the actor minimises
    alpha log pi(a~|s) - min Q(s, a~) with a~ = tanh(z(s) + sigma eps); soft target updates.
    Returns the device stats (critic 1 [4], critic 2 [4], actor [4])."""
    import torch
    x, xn, a = batch["x"], batch["x_next"], batch["a"]
    B, S, K = int(x.shape[0]), int(x.shape[1]), int(a.shape[1])
    H = max(actor.dims[1], actor.dims[2])
    # target: a' and log pi(a'|s') from the current actor, min of the target critics
    zn = _zeros((B, K), torch.float32)
    actor.forward(xn, zn, stream=stream)
    an = _zeros((B, K), torch.float32)
    lpn = _zeros(B, torch.float32)
    fin.fin_squash(zn, an, eps=batch["eps_next"], logp=lpn, sigma=sigma, stream=stream)
    xan = _zeros((B, S + K), torch.float32)
    fin.fin_concat_obs_action(xn, an, xan, stream=stream)
    qn = [_zeros((B, 1), torch.float32) for _ in range(2)]
    for c, q in zip(critics_targ, qn):
        c.forward(xan, q, stream=stream)
    st_c = [_critic_step(c, x, a, S, batch, qn[0].view(-1), qn[1].view(-1), lpn, gamma, alpha, lr_critic, stream)
            for c in critics]
    # actor on the reparameterised sample
    z = _zeros((B, K), torch.float32)
    hid = _zeros((B, 2, H), torch.int16)
    actor.forward(x, z, hid, stream=stream)
    at = _zeros((B, K), torch.float32)
    lp = _zeros(B, torch.float32)
    fin.fin_squash(z, at, eps=batch["eps"], logp=lp, sigma=sigma, stream=stream)
    (q1, g1), (q2, g2) = (_q_and_dq(c, x, at, S, stream) for c in critics)
    gz = _zeros((B, K), torch.float32)
    st_a = _zeros(4, torch.float64)
    fin.fin_actor_head(at, q1, g1[:, S:], gz, st_a, logp=lp, q2=q2, dq2=g2[:, S:], alpha=alpha, stream=stream)
    fin.fin_policy_backward(x, hid, gz, actor.w[1], actor.w[2], actor.grads, stream=stream)
    actor.adam(lr_actor, stream=stream)
    actor.load(stream=stream)
    for t, c in zip(critics_targ, critics):
        t.soft_update_from(c, tau, stream=stream)
    return st_c[0], st_c[1], st_a


def value_update(vnet: DenseNet, x, returns, lr: float = 3e-4, stream=None):
    """The PPO member's value regression (the value MSE of its loss; reading R-AC's
    critic head with gamma = 0, so y = the GAE return R): V(s) a float32 DenseNet on the widened
    observation, L_V = mean (V(s) - R)^2, one Adam step.  Returns the device stats [4] (L, mean V,
    mean R, B)."""
    import torch
    B, S = int(x.shape[0]), int(x.shape[1])
    xf = _zeros((B, S), torch.float32)
    fin.fin_concat_obs_action(x, None, xf, stream=stream)
    hid = _zeros((B, vnet.dims[1] + vnet.dims[2]), torch.float32)
    v = _zeros((B, 1), torch.float32)
    vnet.forward(xf, v, hid, stream=stream)
    g = _zeros(B, torch.float32)
    st = _zeros(4, torch.float64)
    zero = _zeros(B, torch.uint8)
    fin.fin_critic_head(v.view(-1), returns, zero, returns, g, st, gamma=0.0, alpha=0.0, stream=stream)
    fin.fin_dense_backward(xf, hid, g.view(B, 1), vnet.weights(), grads=vnet.grads, stream=stream)
    vnet.adam(lr, stream=stream)
    return st
