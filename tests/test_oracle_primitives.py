"""Pins for the oracle's primitives (CPU only): Philox, index map, stacking, layers.

Each test checks oracle/ against something other than itself: published
known-answer vectors, an independent Philox (synth/), Python big-integer
arithmetic, hand-tabulated fixtures (tests/golden/), torch CPU library
routines in fp64, closed forms and finite differences.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_philox_known_answers():
    for case in _gold("philox_kat.json")["cases"]:
        ctr = [int(x, 16) for x in case["ctr"]]
        key = [int(x, 16) for x in case["key"]]
        out = [int(x, 16) for x in case["out"]]
        assert list(O.philox(ctr, key)) == out


def test_index_map_against_bigint_and_independent_philox():
    # u is the 64-bit word of an independent Philox (synth); tau = base + floor(u*M/2^64)
    seed, learner, rnd, B = 1507, 3, (1 << 33) + 17, 33
    n, size = 123_456, 100_000
    tau = O.sample_indices(n, size, B, seed, learner, rnd)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for i in range(B):
        x = synth.philox([i // 2, learner, rnd & 0xFFFFFFFF, ((rnd >> 32) & 0xFFFFFF) | (3 << 24)], key)
        u = int(x[0]) | (int(x[1]) << 32) if i % 2 == 0 else int(x[2]) | (int(x[3]) << 32)
        assert tau[i] == (n - size) + (u * (size - 1) >> 64)


def test_index_range_and_forced_outcome():
    # one valid transition (size 2): every draw is slot n-size
    assert set(O.sample_indices(2, 2, 4, 1, 0, 0)) == {0}
    with pytest.raises(ValueError):
        O.sample_indices(1, 1, 4, 1, 0, 0)  # no valid transition: not ready
    # wrapped ring: tau in [n-size, n-2]
    for rnd in range(20):
        t = O.sample_indices(50, 8, 64, 7, 1, rnd)
        assert t.min() >= 42 and t.max() <= 48


def test_index_uniformity_chi_square():
    from scipy.stats import chisquare
    M = 1000
    draws = np.concatenate([O.sample_indices(M + 1, M + 1, 1000, 1507, 0, k) for k in range(100)])
    hist = np.bincount(draws, minlength=M)
    assert hist.size == M
    assert chisquare(hist).pvalue > 0.01


def test_index_deterministic_and_learner_distinct():
    a = O.sample_indices(10_000, 10_000, 32, 1507, 0, 5)
    b = O.sample_indices(10_000, 10_000, 32, 1507, 0, 5)
    c = O.sample_indices(10_000, 10_000, 32, 1507, 1, 5)
    assert (a == b).all() and not (a == c).all()


def _ring8():
    g = _gold("stack_ring8.json")
    ring = O.Ring(g["C"])
    for t in range(g["n"]):
        fr = np.full((1, 84, 84), 10 * (t + 1), np.uint8)
        ring.insert(fr, [0], [0.0], [1 if t in g["terminal_steps"] else 0])
    return ring, g


def test_stacking_hand_table():
    ring, g = _ring8()
    assert ring.n == g["n"] and ring.size == g["C"]
    for t, expect in g["stacks"].items():
        st = ring.stack(int(t))
        for c in range(4):
            assert (st[c] == expect[c]).all(), (t, c)


def test_gather_pairs_s_and_next_state():
    ring, g = _ring8()
    tau = np.arange(g["valid_tau"][0], g["valid_tau"][1] + 1)
    s, s2, a, r, d = ring.gather(tau)
    for i, t in enumerate(tau):
        assert (s[i] == ring.stack(t)).all() and (s2[i] == ring.stack(t + 1)).all()
        assert d[i] == (1 if t in g["terminal_steps"] else 0)


def test_ring_eviction_fifo():
    # capacity 3, insert a,b,c,d -> b,c,d
    ring = O.Ring(3)
    for v in (1, 2, 3, 4):
        ring.insert(np.full((1, 84, 84), v, np.uint8), [v], [float(v)], [0])
    assert sorted(ring.frames[:, 0, 0].tolist()) == [2, 3, 4]
    assert ring.size == 3 and ring.n == 4


def test_round_bf16_matches_torch_rne():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32),
                        np.float32([1.0, 1.00390625, 1.01171875, -3.0e-5, 65504.0])])
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    got = np.array([O.round_bf16(float(v)) for v in x])
    assert (got == ref).all()


@pytest.mark.parametrize("B,Cin,H,Cout,k,s", [(2, 3, 11, 5, 3, 2), (1, 4, 84, 32, 8, 4), (2, 32, 20, 64, 4, 2),
                                             (3, 64, 9, 64, 3, 1)])
def test_conv_forward_matches_torch(B, Cin, H, Cout, k, s):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((B, Cin, H, H))
    w = rng.standard_normal((Cout, Cin, k, k))
    b = rng.standard_normal(Cout)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), torch.from_numpy(b), stride=s)
    assert np.allclose(O.conv2d_fwd(x, w, b, s), ref.numpy(), rtol=1e-12, atol=1e-12)


def test_conv_forward_special_cases():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 3, 12, 12))
    # zero weights -> bias only (SPEC S:48 analogue)
    y = O.conv2d_fwd(x, np.zeros((4, 3, 4, 4)), np.arange(4.0), 2)
    assert (y == np.arange(4.0)[None, :, None, None]).all()
    # one-hot kernel at (c=1, ky=2, kx=1) with stride 2 -> strided crop of channel 1
    w = np.zeros((1, 3, 4, 4))
    w[0, 1, 2, 1] = 1.0
    y = O.conv2d_fwd(x, w, None, 2)
    assert (y[:, 0] == x[:, 1, 2:2 + 2 * 5:2, 1:1 + 2 * 5:2]).all()


def test_linear_matches_closed_form():
    rng = np.random.default_rng(3)
    x, w, b = rng.standard_normal((5, 7)), rng.standard_normal((3, 7)), rng.standard_normal(3)
    assert np.allclose(O.linear_fwd(x, w, b), x @ w.T + b, rtol=1e-13, atol=1e-13)
    dy = rng.standard_normal((5, 3))
    assert np.allclose(O.linear_bwd_data(dy, w), dy @ w, rtol=1e-13, atol=1e-13)
    dw, db = O.linear_bwd_weight(dy, x)
    assert np.allclose(dw, dy.T @ x, rtol=1e-13, atol=1e-13) and np.allclose(db, dy.sum(0))
    # single linear layer, one-hot upstream u on row a -> grad row a = u*x, bias u
    u = np.zeros((1, 3))
    u[0, 1] = 0.7
    dw, db = O.linear_bwd_weight(u, x[:1])
    assert np.allclose(dw[1], 0.7 * x[0]) and (dw[[0, 2]] == 0).all() and np.allclose(db, [0, 0.7, 0])


@pytest.mark.parametrize("B,Cin,H,Cout,k,s", [(2, 3, 11, 5, 3, 2), (2, 32, 20, 64, 4, 2), (2, 64, 9, 64, 3, 1)])
def test_conv_backward_matches_torch_autograd(B, Cin, H, Cout, k, s):
    rng = np.random.default_rng(4)
    x = torch.from_numpy(rng.standard_normal((B, Cin, H, H))).requires_grad_()
    w = torch.from_numpy(rng.standard_normal((Cout, Cin, k, k))).requires_grad_()
    b = torch.from_numpy(rng.standard_normal(Cout)).requires_grad_()
    y = torch.nn.functional.conv2d(x, w, b, stride=s)
    dy = torch.from_numpy(rng.standard_normal(tuple(y.shape)))
    y.backward(dy)
    dx = O.conv2d_bwd_data(dy.numpy(), w.detach().numpy(), (H, H), s)
    dw, db = O.conv2d_bwd_weight(dy.numpy(), x.detach().numpy(), k, s)
    assert np.allclose(dx, x.grad.numpy(), rtol=1e-11, atol=1e-11)
    assert np.allclose(dw, w.grad.numpy(), rtol=1e-11, atol=1e-11)
    assert np.allclose(db, b.grad.numpy(), rtol=1e-11, atol=1e-11)


def test_conv_backward_finite_differences_tiny_net():
    # tiny conv -> relu -> conv net; all coordinates; central FD, h=1e-6
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 2, 9, 9))
    w1, b1 = rng.standard_normal((3, 2, 3, 3)), rng.standard_normal(3)
    w2, b2 = rng.standard_normal((2, 3, 2, 2)), rng.standard_normal(2)
    up = rng.standard_normal((2, 2, 3, 3))

    def f(w1_, b1_):
        z = O.conv2d_fwd(x, w1_, b1_, 2)
        return float((O.conv2d_fwd(np.maximum(z, 0), w2, b2, 1) * up).sum()), z

    _, z = f(w1, b1)
    g2 = O.conv2d_bwd_data(up, w2, z.shape[2:], 1) * (z > 0)
    dw1, db1 = O.conv2d_bwd_weight(g2, x, 3, 2)
    assert np.abs(z).min() > 1e-4  # no kink within the FD step
    h = 1e-6
    for idx in np.ndindex(w1.shape):
        wp, wm = w1.copy(), w1.copy()
        wp[idx] += h
        wm[idx] -= h
        fd = (f(wp, b1)[0] - f(wm, b1)[0]) / (2 * h)
        assert abs(fd - dw1[idx]) <= 1e-5 * max(1.0, abs(fd))
    for o in range(3):
        bp, bm = b1.copy(), b1.copy()
        bp[o] += h
        bm[o] -= h
        fd = (f(w1, bp)[0] - f(w1, bm)[0]) / (2 * h)
        assert abs(fd - db1[o]) <= 1e-5 * max(1.0, abs(fd))
