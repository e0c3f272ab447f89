"""Pins for oracle/quant.py, oracle/mlp.py and oracle/policy.py -- CPU only."""
import math
import struct

import numpy as np
import pytest
import torch

from oracle import mlp, policy, quant, rollout
from synth import policy as spol


def _f32_to_bf16_value(x: float) -> float:
    """Independent pin: float32 -> bf16 RNE on the bit pattern (textbook round-bias trick)."""
    (u,) = struct.unpack("<I", struct.pack("<f", x))
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    (v,) = struct.unpack("<f", struct.pack("<I", u))
    return v


def test_bf16_exact_cases():
    assert quant.bf16(1.0) == 1.0
    assert quant.bf16(1.0 + 2 ** -8) == 1.0                 # tie -> even (down)
    assert quant.bf16(1.0 + 3 * 2 ** -8) == 1.0 + 2 ** -6   # tie -> even (up)
    assert quant.bf16(1.0 + 2 ** -8 + 2 ** -40) == 1.0 + 2 ** -7   # just above the tie
    assert quant.bf16(-2.5) == -2.5
    assert quant.bf16(3.0e38) == math.inf or quant.bf16(3.0e38) > 3e38
    assert quant.bf16(0.0) == 0.0


def test_bf16_matches_float32_path_on_float32_values():
    """For inputs exactly representable in float32 a single f32->bf16 RNE must agree."""
    rng = np.random.default_rng(0)
    xs = rng.standard_normal(3000).astype(np.float32) * np.float32(7.0)
    for x in xs:
        assert quant.bf16(float(x)) == _f32_to_bf16_value(float(x))
    # torch's float32 -> bfloat16 conversion is RNE as well (library cross-check)
    t = torch.from_numpy(xs).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(t, quant.bf16_fast(xs.astype(np.float64)))


def test_bf16_fast_equals_fraction_version():
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.standard_normal(4000) * 10 ** rng.uniform(-6, 6, 4000),
                        # exact ties and near-ties of the bf16 grid
                        (1 + (2 * rng.integers(0, 128, 500) + 1) * 2.0 ** -8) * 2.0 ** rng.integers(-20, 20, 500),
                        np.array([1e-40, -3e-39, 0.0, -0.0])])
    fast = quant.bf16_fast(x)
    slow = np.array([quant.bf16(float(v)) for v in x])
    assert np.array_equal(fast, slow)


def test_rha():
    assert quant.rha(2.5) == 3 and quant.rha(-2.5) == -3 and quant.rha(0.49999999999999994) == 0
    assert quant.rha(-0.5) == -1 and quant.rha(1.4999) == 1 and quant.rha(100.0) == 100


def _rand_layers(dims, seed):
    return spol.random_bias(spol.kaiming_bf16(dims, seed), seed + 100)


def test_forward_matches_explicit_loops():
    layers = mlp.layers_f64(_rand_layers((13, 9, 7, 5), 3))
    rng = np.random.default_rng(4)
    X = rng.standard_normal((6, 13))
    z = mlp.forward(layers, X)
    for i in range(6):
        zl = mlp.forward_loops(layers, X[i])
        np.testing.assert_allclose(z[i], zl, rtol=1e-12, atol=1e-12)


def test_forward_library_cross_check_torch_linear():
    layers = mlp.layers_f64(_rand_layers((301, 256, 256, 30), 0))
    rng = np.random.default_rng(5)
    X = rng.standard_normal((16, 301))
    h = torch.from_numpy(quant.bf16_fast(X))
    for li, (w, b) in enumerate(layers):
        z = torch.nn.functional.linear(h, torch.from_numpy(w), torch.from_numpy(b))
        h = torch.from_numpy(quant.bf16_fast(torch.relu(z).numpy())) if li < 2 else z
    np.testing.assert_allclose(mlp.forward(layers, X), h.numpy(), rtol=1e-12, atol=1e-12)


def test_zero_weights_give_bias_and_identity_layer():
    L = [(np.zeros((4, 3)), np.zeros(4)), (np.zeros((2, 4)), np.array([0.5, -1.25]))]
    assert mlp.forward(L, np.ones((1, 3))).tolist() == [[0.5, -1.25]]
    eye = [(np.eye(5), np.zeros(5))]
    x = np.array([[0.5, -2.0, 1.0, 0.25, 3.0]])   # bf16-exact
    assert np.array_equal(mlp.forward(eye, x), x)


def test_dyadic_mlp_is_exact():
    """Dyadic weights / inputs in {0, +-1/2, +-1, +-2} with small fan-in: every
    product and partial sum is exact, so z equals the rational result."""
    rng = np.random.default_rng(6)
    vals = np.array([0.0, 0.5, -0.5, 1.0, -1.0, 2.0, -2.0])
    L = [(rng.choice(vals, (8, 6)), rng.choice(vals, 8)), (rng.choice(vals, (4, 8)), np.zeros(4))]
    x = rng.choice(vals, (5, 6))
    z = mlp.forward(L, x)
    ref = np.maximum(x @ L[0][0].T + L[0][1], 0) @ L[1][0].T
    assert np.array_equal(z, ref)


def test_kaiming_bound_and_bf16():
    layers = spol.kaiming_bf16((301, 256, 256, 30), 0)
    w = mlp.bf16_bits_to_f64(layers[0][0])
    assert w.shape == (256, 301) and np.abs(w).max() <= math.sqrt(6 / 301) * (1 + 2 ** -8)
    assert np.array_equal(quant.bf16_fast(w), w)     # already bf16 values
    assert np.array_equal(spol.kaiming_bf16((301, 256), 0)[0][0], layers[0][0])


def test_sampling_special_cases():
    """eps=0, z=0 -> 0 shares; a=1 -> +100; clipping at +-1."""
    assert policy.shares(policy.gaussian_action(0.0, 0.0)) == 0
    assert policy.shares(1.0) == 100 and policy.shares(-1.0) == -100
    assert policy.gaussian_action(50.0, 5.0) == 1.0 and policy.gaussian_action(-50.0, -5.0) == -1.0
    assert policy.shares(0.005) == 1 and policy.shares(-0.005) == -1   # rha(0.5)
    assert policy.sac_action(0.0, 0.0) == 0.0


def test_ou_closed_form_and_stationary_std():
    x = 1.0
    for t in range(1, 30):
        x = policy.ou_update(x, 0.0)
        assert x == pytest.approx(0.85 ** t, rel=1e-12)
    rng = np.random.default_rng(7)
    xs = np.zeros(65536)
    for t in range(200):
        xs = (xs + 0.15 * (0.0 - xs)) + 0.2 * rng.standard_normal(65536)
    sd = 0.2 / math.sqrt(1 - 0.85 ** 2)                       # = 0.3797
    assert abs(xs.std() - sd) < 3 * sd / math.sqrt(2 * 65536) + 2e-3
    # the oracle's scalar OU gives the same stationary law
    ys = []
    for i in range(4000):
        y = 0.0
        for t in range(60):
            y = policy.ou_update(y, float(rng.standard_normal()))
        ys.append(y)
    assert abs(np.std(ys) - sd) < 0.03


def test_ensemble_unanimity_and_zero():
    """identical members + identical noise -> ensemble action = member action."""
    rng = np.random.default_rng(8)
    for _ in range(500):
        z, e = float(rng.standard_normal()), float(rng.standard_normal())
        a = policy.gaussian_action(z, e)
        sh, abar, _ = rollout.ensemble_shares([0, 0, 0], [[z]] * 3, [[e]] * 3, [0.0])
        if abs(abs(100 * a) % 1.0 - 0.5) > 1e-9:
            assert sh[0] == policy.shares(a)
    sh, abar, ou = rollout.ensemble_shares([0, 1, 2], [[0.0]] * 3, [[0.0]] * 3, [0.0])
    assert sh == [0] and abar == [0.0] and ou == [0.0]


def test_argmax_and_epsilon_greedy():
    assert policy.argmax_lowest([1.0, 3.0, 3.0]) == 1
    assert policy.argmax_lowest([2.0, 2.0, 2.0]) == 0
    assert policy.epsilon_greedy([0.0, 1.0, 0.0], 0.005, 0.004, 0.1) == 0
    assert policy.epsilon_greedy([0.0, 1.0, 0.0], 0.005, 0.006, 0.1) == 1
    assert policy.epsilon_greedy([0.0, 1.0, 0.0], 0.005, 0.0, 0.9999) == 2


def _fp32_device_model(layers64, x):
    """A stand-in 'device': fp32 accumulation, bf16 activations (numpy float32 matmul)."""
    h = quant.bf16_fast(x).astype(np.float32)
    hid = []
    for li, (w, b) in enumerate(layers64):
        z = h @ w.T.astype(np.float32) + b.astype(np.float32)
        if li < len(layers64) - 1:
            a = quant.bf16_fast(np.maximum(z, 0).astype(np.float64))
            hid.append(spol.f64_to_bf16_bits(a))
            h = a.astype(np.float32)
        else:
            out = z.astype(np.float64)
    return np.stack(hid, axis=1), out


def test_teacher_forced_layers_accepts_fp32_and_rejects_corruption():
    layers = mlp.layers_f64(_rand_layers((301, 256, 256, 30), 11))
    rng = np.random.default_rng(12)
    x = rng.standard_normal((64, 301)) * 2
    hid, z = _fp32_device_model(layers, x)
    amb, tot = mlp.teacher_forced_layers(layers, x, hid, z)
    assert tot == 64 * 512 and amb < tot * 1e-2
    bad = hid.copy()
    i, j = np.argwhere(bad[:, 0, :] != 0)[0]
    bad[i, 0, j] += 2                                   # two bf16 ulps off
    with pytest.raises(AssertionError):
        mlp.teacher_forced_layers(layers, x, bad, z)
    zb = z.copy()
    zb[3, 4] += 1e-3
    with pytest.raises(AssertionError):
        mlp.teacher_forced_layers(layers, x, hid, zb)
    # an observation-encoding error (input not what the oracle encodes) is caught at layer 1
    with pytest.raises(AssertionError):
        mlp.teacher_forced_layers(layers, x * 1.01, hid, z)


def test_ambiguous_rows_and_row_mask():
    """oracle.mlp.ambiguous_rows flags exactly the rows where a hidden pre-activation sits
    within the fp32 bound of a bf16 rounding decision: a 1-input identity-like net whose
    pre-activation is the midpoint between two bf16 neighbours is flagged, one on a bf16
    value is not.  teacher_forced_layers(row_mask=True) marks the rows it accepted an
    ambiguous activation in, and only those."""
    one = 1.0
    mid = 1.0 + 2.0 ** -8              # halfway between bf16 1.0 and 1.0 + 2^-7
    w1 = np.array([[one]])
    layers = [(w1, np.zeros(1)), (np.array([[one]]), np.zeros(1))]
    x = np.array([[1.0], [1.0]])
    # move row 0's pre-activation to the midpoint via the bias (x = 1 exactly in bf16)
    layers_mid = [(w1, np.array([mid - 1.0])), layers[1]]
    rows = mlp.ambiguous_rows(layers_mid, x)
    assert rows.all()
    assert not mlp.ambiguous_rows(layers, x).any()
    # row mask: a device that rounded row 1's midpoint up (legal) is flagged in row 1 only
    hid = np.zeros((2, 2, 1), dtype=np.uint16)
    lo_bits, hi_bits = spol.f64_to_bf16_bits(np.array([1.0, 1.0 + 2.0 ** -7]))
    hid[0, 0, 0], hid[1, 0, 0] = lo_bits, hi_bits      # RNE of the midpoint is 1.0 (even)
    z = np.array([[1.0], [1.0 + 2.0 ** -7]])
    amb, tot, mask = mlp.teacher_forced_layers(layers_mid, x, hid, z, row_mask=True)
    assert amb == 1 and mask.tolist() == [False, True]
