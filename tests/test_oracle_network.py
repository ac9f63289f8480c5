"""Pins for the oracle's Nature-DQN Q-network (§5.1) forward / backward.

References used: the paper's architecture numbers (closed-form shapes and
parameter counts), torch CPU fp64 conv2d/linear + autograd (library routines),
and central finite differences.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
import synth


def test_param_counts_closed_form():
    # conv1 32x(4x8x8), conv2 64x(32x4x4), conv3 64x(64x3x3), fc 512, linear nA; +biases
    for nA in (4, 18):
        expect = (32 * 256 + 32) + (64 * 512 + 64) + (64 * 576 + 64) + (512 * 3136 + 512) + (nA * 512 + nA)
        assert O.param_count(nA) == expect
    assert O.param_count(18) == 1_693_362 and O.param_count(4) == 1_686_180
    # spatial chain 84 -> 20 -> 9 -> 7 (valid convs; 7*7*64 = 3136 only fits valid padding, R18)
    assert (84 - 8) // 4 + 1 == 20 and (20 - 4) // 2 + 1 == 9 and (9 - 3) // 1 + 1 == 7
    assert O.acts_per_sample() == 32 * 400 + 64 * 81 + 64 * 49 + 512


def _torch_net(p, x, mode):
    """Independent composition from torch library routines (fp64)."""
    def q(t):
        return t.to(torch.bfloat16).to(torch.float64) if mode == "bf16" else t

    if mode == "bf16":
        z1 = F.conv2d(x, q(p["W1"]), None, stride=4) * float(np.float32(1.0 / 255.0)) + p["b1"][:, None, None]
    else:
        z1 = F.conv2d(x / 255.0, p["W1"], p["b1"], stride=4)
    a1 = q(F.relu(z1))
    a2 = q(F.relu(F.conv2d(a1, q(p["W2"]), p["b2"], stride=2)))
    a3 = q(F.relu(F.conv2d(a2, q(p["W3"]), p["b3"], stride=1)))
    a4 = F.relu(F.linear(a3.reshape(a3.shape[0], -1), q(p["W4"]), p["b4"]))  # a4 stays unrounded (R16)
    return F.linear(a4, p["W5"], p["b5"])


def _inputs(nA, B, seed=0):
    theta = synth.theta0(nA).astype(np.float64)
    rng = np.random.default_rng(seed)
    theta[O.param_count(nA) - nA:] += rng.standard_normal(nA) * 0.1  # non-trivial fc5 bias
    s = rng.integers(0, 256, size=(B, 4, 84, 84), dtype=np.uint8)
    return theta, s


@pytest.mark.parametrize("mode", ["exact", "bf16"])
def test_qnet_forward_matches_torch(mode):
    nA, B = 18, 3
    theta, s = _inputs(nA, B)
    Q, _ = O.qnet_forward(theta, s, nA, mode)
    p = {k: torch.from_numpy(v.copy()) for k, v in O.unflatten(theta, nA).items()}
    ref = _torch_net(p, torch.from_numpy(s.astype(np.float64)), mode).numpy()
    tol = 1e-12 if mode == "exact" else 1e-9  # bf16: rare rounding-boundary flips from summation order
    assert np.max(np.abs(Q - ref)) <= tol * max(1.0, np.max(np.abs(ref)))


def test_qnet_zero_weights_give_bias():
    nA, B = 4, 2
    theta = np.zeros(O.param_count(nA))
    theta[-nA:] = [1.0, -2.0, 0.5, 3.0]
    s = np.random.default_rng(1).integers(0, 256, size=(B, 4, 84, 84), dtype=np.uint8)
    Q, _ = O.qnet_forward(theta, s, nA)
    assert (Q == np.array([1.0, -2.0, 0.5, 3.0])).all()


@pytest.mark.parametrize("mode", ["exact", "bf16"])
def test_qnet_backward_matches_torch_autograd(mode):
    nA, B = 18, 2
    theta, s = _inputs(nA, B, seed=3)
    rng = np.random.default_rng(4)
    dQ = rng.standard_normal((B, nA))
    Q, acts = O.qnet_forward(theta, s, nA, mode)
    G = O.qnet_backward(theta, s, acts, dQ, nA, mode)
    p = {k: torch.from_numpy(v.copy()).requires_grad_() for k, v in O.unflatten(theta, nA).items()}
    if mode == "exact":
        Qt = _torch_net(p, torch.from_numpy(s.astype(np.float64)), mode)
        Qt.backward(torch.from_numpy(dQ))
    else:
        # bf16 contract: gradients flow through the rounded weights and activations unchanged
        # (straight-through), and each backward activation gradient is rounded to bf16.
        class RoundSTE(torch.autograd.Function):
            @staticmethod
            def forward(ctx, t):
                return t.to(torch.bfloat16).to(torch.float64)

            @staticmethod
            def backward(ctx, g):
                return g

        class RoundGrad(torch.autograd.Function):
            @staticmethod
            def forward(ctx, t):
                return t.clone()

            @staticmethod
            def backward(ctx, g):
                return g.to(torch.bfloat16).to(torch.float64)

        x = torch.from_numpy(s.astype(np.float64))
        z1 = F.conv2d(x, RoundSTE.apply(p["W1"]), None, stride=4) * float(np.float32(1 / 255.0)) + \
            p["b1"][:, None, None]
        a1 = RoundGrad.apply(RoundSTE.apply(F.relu(z1)))
        a2 = RoundGrad.apply(RoundSTE.apply(F.relu(F.conv2d(a1, RoundSTE.apply(p["W2"]), p["b2"], stride=2))))
        a3 = RoundGrad.apply(RoundSTE.apply(F.relu(F.conv2d(a2, RoundSTE.apply(p["W3"]), p["b3"], stride=1))))
        a4 = RoundGrad.apply(F.relu(F.linear(a3.reshape(B, -1), RoundSTE.apply(p["W4"]), p["b4"])))
        Qt = F.linear(a4, p["W5"], p["b5"])
        Qt.backward(torch.from_numpy(dQ))
    ref = np.concatenate([p[k].grad.numpy().ravel() for k, _ in O.param_shapes(nA)])
    off = 0
    for name, shp in O.param_shapes(nA):
        n = int(np.prod(shp))
        g, r = G[off:off + n], ref[off:off + n]
        err = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)
        assert err < (1e-11 if mode == "exact" else 1e-6), (name, err)
        off += n


def test_qnet_backward_finite_differences_nature_shape():
    # >= 200 random coordinates across all 10 tensors, central FD in fp64
    nA, B = 4, 1
    theta, s = _inputs(nA, B, seed=6)
    rng = np.random.default_rng(7)
    dQ = rng.standard_normal((B, nA))
    Q, acts = O.qnet_forward(theta, s, nA)
    G = O.qnet_backward(theta, s, acts, dQ, nA)

    def f(th):
        return float((O.qnet_forward(th, s, nA)[0] * dQ).sum())

    h = 1e-6
    off, checked = 0, 0
    for name, shp in O.param_shapes(nA):
        n = int(np.prod(shp))
        for i in rng.choice(n, size=min(n, 24), replace=False):
            tp, tm = theta.copy(), theta.copy()
            tp[off + i] += h
            tm[off + i] -= h
            fd = (f(tp) - f(tm)) / (2 * h)
            assert abs(fd - G[off + i]) <= 1e-5 * max(abs(fd), 1e-3), (name, i, fd, G[off + i])
            checked += 1
        off += n
    assert checked >= 200


def test_zero_upstream_gives_zero_gradient():
    nA, B = 4, 2
    theta, s = _inputs(nA, B, seed=8)
    _, acts = O.qnet_forward(theta, s, nA)
    assert (O.qnet_backward(theta, s, acts, np.zeros((B, nA)), nA) == 0).all()
