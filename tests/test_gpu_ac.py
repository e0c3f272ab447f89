"""GPU parity of the DDPG / SAC update pieces (reading R-AC) against
oracle/learn.py: the critic forward / backward (fp32 contractions vs float64, the backward teacher
forced on the device's own hidden activations), the float64 heads (to the last f32 ulp), the soft
update (bit for bit), and one full DDPG and SAC update through paper_2501_10709_b200.learner."""
import numpy as np
import pytest

from gpu_util import dev, host, needs_gpu, zeros
from oracle import learn as olearn

pytestmark = [pytest.mark.gpu, needs_gpu]

S, K = 301, 30
CRITIC = (S + K, 256, 256, 1)


def _close(g, o, rel=1e-4, scale=2e-5):
    """fp32 contraction vs float64: |g - o| <= scale max|o| + rel |o|."""
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    bad = np.abs(g - o) > scale * np.abs(o).max() + rel * np.abs(o)
    assert not bad.any(), (int(bad.sum()), float(np.abs(g - o).max()), float(np.abs(o).max()))


def _ulps(g, o, n=1):
    """float64 head rounded to f32 on the device vs the oracle's float64: within n f32 ulps."""
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    tol = n * np.spacing(np.abs(o).astype(np.float32)).astype(np.float64) + 1e-45
    assert np.all(np.abs(g - o) <= tol), float(np.max(np.abs(g - o) / tol))


def _critic(seed):
    from paper_2501_10709_b200.learner import DenseNet
    return DenseNet(CRITIC, seed)


def _obs(rng, B):
    from synth import policy as spol
    return spol.f64_to_bf16_bits(rng.standard_normal((B, S)))


def _layers64(net):
    return [(host(w).astype(np.float64), host(b).astype(np.float64)) for w, b in net.layers]


@pytest.mark.parametrize("B", [1000, 65, 1])
def test_dense_forward_backward_matches_oracle(B):
    """The critic on [x; a] (331-256-256-1): fin_concat_obs_action exact; forward within fp32
    accumulation of the float64 forward; backward (parameter gradients and dQ/dx) against
    dense_backward_np fed with the device's hidden activations."""
    import torch
    from paper_2501_10709_b200 import fin
    from oracle import mlp as omlp
    rng = np.random.default_rng(B)
    net = _critic(3)
    xb = _obs(rng, B)
    a = rng.uniform(-1, 1, (B, K)).astype(np.float32)
    xa = zeros((B, S + K), torch.float32)
    fin.fin_concat_obs_action(dev(xb.view(np.int16)), dev(a), xa)
    xo = np.concatenate([omlp.bf16_bits_to_f64(xb), a.astype(np.float64)], axis=1)
    assert np.array_equal(host(xa).astype(np.float64), xo)
    hid = zeros((B, 512), torch.float32)
    q = zeros((B, 1), torch.float32)
    net.forward(xa, q, hid)
    L64 = _layers64(net)
    h1, h2, out = olearn.dense_forward(L64, xo)
    _close(host(hid)[:, :256], h1)
    _close(host(hid)[:, 256:], h2)
    _close(host(q), out)
    g = rng.standard_normal((B, 1)).astype(np.float32)
    gx = zeros((B, S + K), torch.float32)
    fin.fin_dense_backward(xa, hid, dev(g), net.weights(), grads=net.grads, g_x=gx)
    hd = host(hid).astype(np.float64)
    ref, rgx = olearn.dense_backward_np(L64, xo, hd[:, :256], hd[:, 256:], g.astype(np.float64))
    for (dw, db), (rw, rb) in zip(net.grads, ref):
        _close(host(dw), rw)
        _close(host(db), rb)
    _close(host(gx), rgx)
    # only the input gradient (the actor's dQ/da path)
    gx2 = zeros((B, S + K), torch.float32)
    fin.fin_dense_backward(xa, hid, dev(g), net.weights(), g_x=gx2)
    assert np.array_equal(host(gx2), host(gx))


def test_dense_forward_paper_critic_multi_output():
    """A second shape (the paper's 64-32 widths, 3 outputs, ragged 64-row tiles)."""
    import torch
    from paper_2501_10709_b200 import fin
    from paper_2501_10709_b200.learner import DenseNet
    rng = np.random.default_rng(8)
    net = DenseNet((37, 64, 32, 3), 5)
    B = 333
    x = rng.standard_normal((B, 37)).astype(np.float32)
    hid = zeros((B, 96), torch.float32)
    out = zeros((B, 3), torch.float32)
    net.forward(dev(x), out, hid)
    L64 = _layers64(net)
    h1, h2, o = olearn.dense_forward(L64, x.astype(np.float64))
    _close(host(out), o)
    g = rng.standard_normal((B, 3)).astype(np.float32)
    gx = zeros((B, 37), torch.float32)
    fin.fin_dense_backward(dev(x), hid, dev(g), net.weights(), grads=net.grads, g_x=gx)
    hd = host(hid).astype(np.float64)
    ref, rgx = olearn.dense_backward_np(L64, x.astype(np.float64), hd[:, :64], hd[:, 64:], g.astype(np.float64))
    for (dw, db), (rw, rb) in zip(net.grads, ref):
        _close(host(dw), rw)
        _close(host(db), rb)
    _close(host(gx), rgx)


def test_squash_matches_oracle():
    """a = tanh(z + sigma eps) to 1 f32 ulp and log pi to 2 ulps, including saturated |u| up to 40
    (the stable log(1 - tanh^2)); DDPG's tanh z (no eps)."""
    import torch
    from paper_2501_10709_b200 import fin
    rng = np.random.default_rng(4)
    B = 500
    z = rng.normal(0, 2, (B, K)).astype(np.float32)
    z[:5] = rng.uniform(-40, 40, (5, K))
    eps = rng.standard_normal((B, K)).astype(np.float32)
    a, lp = zeros((B, K), torch.float32), zeros(B, torch.float32)
    fin.fin_squash(dev(z), a, eps=dev(eps), logp=lp, sigma=0.1)
    oa, olp = olearn.squash(z.astype(np.float64).tolist(), eps.astype(np.float64).tolist(), 0.1)
    _ulps(host(a), np.array(oa))
    _ulps(host(lp), np.array(olp), 2)
    assert np.isfinite(host(lp)).all()
    a2 = zeros((B, K), torch.float32)
    fin.fin_squash(dev(z), a2)
    oa2, _ = olearn.squash(z.astype(np.float64).tolist())
    _ulps(host(a2), np.array(oa2))
    with pytest.raises(fin.FinError):
        fin.fin_squash(dev(z), a2, logp=lp)           # a density needs eps


@pytest.mark.parametrize("variant", ["ddpg", "sac"])
def test_critic_head_matches_oracle(variant):
    import torch
    from paper_2501_10709_b200 import fin
    rng = np.random.default_rng(9)
    B = 777
    q, r, q1n, q2n, lpn = (rng.standard_normal(B).astype(np.float32) for _ in range(5))
    done = (rng.random(B) < 0.2).astype(np.uint8)
    sac = variant == "sac"
    g, st = zeros(B, torch.float32), zeros(4, torch.float64)
    fin.fin_critic_head(dev(q), dev(r), dev(done), dev(q1n), g, st, q2_next=dev(q2n) if sac else None,
                        logp_next=dev(lpn) if sac else None, gamma=0.99, alpha=0.2)
    f = lambda v: v.astype(np.float64)
    y = olearn.critic_targets(f(r), done, f(q1n), 0.99, f(q2n) if sac else None, f(lpn) if sac else None, 0.2)
    L, og = olearn.critic_head(f(q), y)
    _ulps(host(g), np.array(og))
    s = host(st)
    assert s[0] == pytest.approx(L, rel=1e-12) and s[2] == pytest.approx(np.mean(y), rel=1e-12, abs=1e-14)
    assert s[1] == pytest.approx(np.mean(f(q)), rel=1e-12, abs=1e-14) and s[3] == B


@pytest.mark.parametrize("variant", ["ddpg", "sac"])
def test_actor_head_matches_oracle(variant):
    """dq taken as row views of a wider [B][S + K] tensor (the critic's g_x), as the learner does."""
    import torch
    from paper_2501_10709_b200 import fin
    rng = np.random.default_rng(12)
    B = 640
    a = np.tanh(rng.normal(0, 1, (B, K))).astype(np.float32)
    lp = rng.normal(-20, 5, B).astype(np.float32)
    q1, q2 = rng.standard_normal(B).astype(np.float32), rng.standard_normal(B).astype(np.float32)
    gx1 = rng.standard_normal((B, S + K)).astype(np.float32)
    gx2 = rng.standard_normal((B, S + K)).astype(np.float32)
    d1, d2 = dev(gx1), dev(gx2)
    gz, st = zeros((B, K), torch.float32), zeros(4, torch.float64)
    f = lambda v: v.astype(np.float64)
    if variant == "ddpg":
        fin.fin_actor_head(dev(a), dev(q1), d1[:, S:], gz, st)
        L, og = olearn.ddpg_actor_head(f(a).tolist(), f(q1), f(gx1[:, S:]).tolist())
    else:
        fin.fin_actor_head(dev(a), dev(q1), d1[:, S:], gz, st, logp=dev(lp), q2=dev(q2), dq2=d2[:, S:], alpha=0.2)
        L, og = olearn.sac_actor_head(f(a).tolist(), f(lp), f(q1), f(gx1[:, S:]).tolist(), f(q2),
                                      f(gx2[:, S:]).tolist(), 0.2)
    _ulps(host(gz), np.array(og))
    assert host(st)[0] == pytest.approx(L, rel=1e-12) and host(st)[3] == B


def test_soft_update_bitwise():
    import torch
    from paper_2501_10709_b200 import fin
    rng = np.random.default_rng(2)
    n = 100003
    t, o = rng.standard_normal(n).astype(np.float32), rng.standard_normal(n).astype(np.float32)
    for tau in (0.005, 1.0, 0.0, 0.3):
        td = dev(t)
        fin.fin_soft_update(td, dev(o), tau)
        assert np.array_equal(host(td), olearn.soft_update(t, o, tau)), tau


def _batch(rng, B, sac):
    r = rng.standard_normal(B).astype(np.float32)
    b = dict(x=dev(_obs(rng, B).view(np.int16)), x_next=dev(_obs(rng, B).view(np.int16)),
             a=dev(np.tanh(rng.normal(0, 1, (B, K))).astype(np.float32)), reward=dev(r),
             done=dev((rng.random(B) < 0.1).astype(np.uint8)))
    if sac:
        b["eps"] = dev(rng.standard_normal((B, K)).astype(np.float32))
        b["eps_next"] = dev(rng.standard_normal((B, K)).astype(np.float32))
    return b


def _critic_loss(net, batch, y):
    import torch
    from paper_2501_10709_b200 import fin
    B = int(batch["x"].shape[0])
    xa = zeros((B, S + K), torch.float32)
    fin.fin_concat_obs_action(batch["x"], batch["a"], xa)
    q = zeros((B, 1), torch.float32)
    net.forward(xa, q)
    return float(np.mean((host(q)[:, 0].astype(np.float64) - y) ** 2))


@pytest.mark.parametrize("variant", ["ddpg", "sac"])
def test_update_end_to_end(variant):
    """One full update through learner.ddpg_update / sac_update on the C1 actor (301-256-256-30) and
    331-256-256-1 critics, B = 1024: the critic statistics equal the oracle's head on the device's
    own forward values (targets from the target nets at s'); one Adam step with a small rate lowers
    each critic's loss at fixed targets; the actor's policy moved and reloads; the targets moved by
    exactly tau of the difference (bitwise, float64 blend); a second update runs."""
    import torch
    from paper_2501_10709_b200 import fin, learner
    from synth import policy as spol
    rng = np.random.default_rng(40)
    B = 1024
    sac = variant == "sac"
    layers = spol.random_bias(spol.kaiming_bf16(spol.STOCK_DIMS, 11), 12)
    kind = fin.FIN_SAC_SQUASH if sac else fin.FIN_DDPG_OU
    actor = learner.Actor(kind, layers)
    batch = _batch(rng, B, sac)
    critics = [_critic(20), _critic(21)] if sac else [_critic(20)]
    targs = [c.copy() for c in critics]
    for t in targs:   # targets differ from the online critics (as after some training)
        for w, _ in t.layers:
            w.mul_(0.9)
    before = [[p.clone() for p in t.params()] for t in targs]
    online_before = [[p.clone() for p in c.params()] for c in critics]
    z0 = zeros((B, K), torch.float32)
    actor.forward(batch["x"], z0)
    # the oracle's targets from the device's own next-state values
    zn = zeros((B, K), torch.float32)
    if sac:
        actor.forward(batch["x_next"], zn)
        an, lpn = olearn.squash(host(zn).astype(np.float64).tolist(), host(batch["eps_next"]).astype(np.float64).tolist(),
                                0.1)
    else:
        actor_targ = learner.Actor(kind, layers)
        actor_targ.forward(batch["x_next"], zn)
        an, lpn = olearn.squash(host(zn).astype(np.float64).tolist())
    xan = zeros((B, S + K), torch.float32)
    fin.fin_concat_obs_action(batch["x_next"], dev(np.array(an, dtype=np.float32)), xan)
    qn = []
    for t in targs:
        q = zeros((B, 1), torch.float32)
        t.forward(xan, q)
        qn.append(host(q)[:, 0].astype(np.float64))
    y = np.array(olearn.critic_targets(host(batch["reward"]).astype(np.float64), host(batch["done"]), qn[0], 0.99,
                                       qn[1] if sac else None, lpn if sac else None, 0.2))
    loss_before = [_critic_loss(c, batch, y) for c in critics]
    if sac:
        stats = learner.sac_update(actor, critics, targs, batch, lr_critic=1e-5, lr_actor=1e-4)
        st_c, st_a = stats[:2], stats[2]
    else:
        stats = learner.ddpg_update(actor, actor_targ, critics[0], targs[0], batch, lr_critic=1e-5, lr_actor=1e-4)
        st_c, st_a = stats[:1], stats[1]
    for st, lb in zip(st_c, loss_before):
        s = host(st)
        assert s[0] == pytest.approx(lb, rel=1e-5) and s[2] == pytest.approx(float(np.mean(y)), rel=1e-5, abs=1e-6)
    for c, lb in zip(critics, loss_before):
        assert _critic_loss(c, batch, y) < lb
    sa = host(st_a)
    assert np.isfinite(sa).all() and sa[3] == B
    z1 = zeros((B, K), torch.float32)
    actor.forward(batch["x"], z1)
    assert not np.array_equal(host(z1), host(z0))
    for t, c, b0 in zip(targs, critics, before):
        for p, o, p0 in zip(t.params(), c.params(), b0):
            assert np.array_equal(host(p), olearn.soft_update(host(p0), host(o), 0.005))
    for c, b0 in zip(critics, online_before):
        assert any(not np.array_equal(host(p), host(p0)) for p, p0 in zip(c.params(), b0))
    if sac:
        learner.sac_update(actor, critics, targs, batch)
    else:
        learner.ddpg_update(actor, actor_targ, critics[0], targs[0], batch)
    torch.cuda.synchronize()


def test_value_update_matches_oracle():
    """PPO's value regression (learner.value_update): V(s) on the widened observation, the squared
    error to the returns (critic head with gamma = 0), its gradient against the oracle's critic_head +
    dense_backward_np on the device's activations (checked before the Adam step), the loss then lower."""
    import torch
    from oracle import mlp as omlp
    from paper_2501_10709_b200 import fin, learner
    rng = np.random.default_rng(50)
    B = 900
    xb = _obs(rng, B)
    x = dev(xb.view(np.int16))
    R = dev(rng.normal(0, 2, B).astype(np.float32))
    v = learner.DenseNet((S, 256, 256, 1), 9)
    xf = zeros((B, S), torch.float32)
    fin.fin_concat_obs_action(x, None, xf)
    assert np.array_equal(host(xf).astype(np.float64), omlp.bf16_bits_to_f64(xb))
    hid = zeros((B, 512), torch.float32)
    out = zeros((B, 1), torch.float32)
    v.forward(xf, out, hid)
    L64 = _layers64(v)
    L0, g = olearn.critic_head(host(out)[:, 0].astype(np.float64), host(R).astype(np.float64))
    hd = host(hid).astype(np.float64)
    ref, _ = olearn.dense_backward_np(L64, omlp.bf16_bits_to_f64(xb), hd[:, :256], hd[:, 256:], np.array(g)[:, None])
    st = learner.value_update(v, x, R, lr=1e-5)
    assert host(st)[0] == pytest.approx(L0, rel=1e-9)
    for (dw, db), (rw, rb) in zip(v.grads, ref):
        _close(host(dw), rw)
        _close(host(db), rb)
    v.forward(xf, out)
    L1, _ = olearn.critic_head(host(out)[:, 0].astype(np.float64), host(R).astype(np.float64))
    assert L1 < L0


def test_learner_contractions_are_deterministic():
    """The split-K contractions sum their partials in a fixed order: two identical calls of the
    critic backward (B = 65,536, split over the batch) and of the PPO gradient give the same bits."""
    import torch
    from paper_2501_10709_b200 import fin
    from paper_2501_10709_b200.learner import DenseNet
    g = torch.Generator(device="cuda").manual_seed(3)
    B = 65536
    net = DenseNet(CRITIC, 7)
    x = torch.randn((B, S + K), device="cuda", generator=g)
    hid = zeros((B, 512), torch.float32)
    out = zeros((B, 1), torch.float32)
    net.forward(x, out, hid)
    go = torch.randn((B, 1), device="cuda", generator=g)
    res = []
    for _ in range(2):
        gx = zeros((B, S + K), torch.float32)
        fin.fin_dense_backward(x, hid, go, net.weights(), grads=net.grads, g_x=gx)
        res.append([host(t).copy() for pair in net.grads for t in pair] + [host(gx)])
    for a, b in zip(*res):
        assert np.array_equal(a, b)


def test_ac_entry_points_reject_bad_arguments():
    """Shape and argument errors are refused before any launch (FIN_E_CONFIG / ValueError)."""
    import torch
    from paper_2501_10709_b200 import fin
    z = zeros((4, K), torch.float32)
    a = zeros((4, K), torch.float32)
    st = zeros(4, torch.float64)
    with pytest.raises(ValueError):
        fin.fin_concat_obs_action(zeros((4, S), torch.int16), zeros((5, K), torch.float32), zeros((4, S + K), torch.float32))
    with pytest.raises(fin.FinError):
        fin.fin_squash(z, a, eps=z, sigma=0.0)
    with pytest.raises(fin.FinError):   # twin critics without log pi (SAC's head needs it)
        fin.fin_actor_head(a, zeros(4, torch.float32), z, zeros((4, K), torch.float32), st, q2=zeros(4, torch.float32),
                           dq2=z)
    with pytest.raises(fin.FinError):
        fin.fin_critic_head(zeros(4, torch.float32), zeros(4, torch.float32), zeros(4, torch.uint8),
                            zeros(4, torch.float32), zeros(4, torch.float32), st, gamma=1.5)
    with pytest.raises(fin.FinError):
        fin.fin_soft_update(zeros(8, torch.float32), zeros(8, torch.float32), tau=2.0)
    with pytest.raises(ValueError):
        fin.fin_dense_forward(zeros((4, 10), torch.float32),
                              [(zeros((8, 9), torch.float32), zeros(8, torch.float32))] * 3, zeros((4, 1), torch.float32))
