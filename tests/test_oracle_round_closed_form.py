"""Closed-form pin of one whole oracle round (the composed learner update + PS apply).

With W1 = 0 every activation of the network is constant over space and over the batch
(valid padding: a constant input plane gives a constant output plane), so Q(s) = Q̂(s')
is one vector, every ReLU mask is fixed per channel and the whole backward (Eq. 2 P:90,
Alg. 1) is a fixed linear map of each sample's dQ_i. This test writes that map out
from the definitions — forward as channel sums of the kernels, each dgrad as the
transposed-correlation definition (scatter of W[o,i,kh,kw]·dz[o,p] to the input position
s·p + (kh,kw)), each wgrad as Σ dz ⊗ input patch — and the first centered-RMSProp step
(reading R2) in its closed form θ⁺ = θ − η g / √(ρ(1−ρ) g² + ε). It shares nothing with the
oracle's loops (oracle.c's 7-loop conv/FC code and gorila_oracle.py's rmsprop_apply) except
the replay gather (pinned by tests/golden/stack_ring8.json) and the sampled τ (pinned by the
Philox KATs), which it reads from the round's info.

A dropped bias term, a transposed operand, a wrong flatten order (R18: fc4 input in (C,H,W)
order), a missing 1/255, a wrong stride in any dgrad, or a wrong sign in TD / the update
fails it.
"""
import numpy as np
import pytest

import oracle as O
import synth


def _convT(W, dz, stride, in_hw):
    """dx[i, s·p + k] += W[o, i, k] · dz[o, p]  (definition of the data gradient of a valid conv)."""
    O_, I_, K, _ = W.shape
    Ho = dz.shape[1]
    dx = np.zeros((I_, in_hw, in_hw))
    span = stride * (Ho - 1) + 1
    for kh in range(K):
        for kw in range(K):
            dx[:, kh:kh + span:stride, kw:kw + span:stride] += np.einsum("oi,ohw->ihw", W[:, :, kh, kw], dz)
    return dx


def constant_activation_params(nA, seed=150704296):
    """θ with W1 = 0 (so every activation plane is constant) and mixed-sign ReLU masks.
    Values are fp32-representable so that the GPU tests can reuse it unchanged."""
    rng = np.random.default_rng(seed)
    p = {
        "W1": np.zeros((32, 4, 8, 8)), "b1": rng.normal(0, 1, 32),
        "W2": rng.normal(0, 0.05, (64, 32, 4, 4)), "b2": rng.normal(0, 0.5, 64),
        "W3": rng.normal(0, 0.05, (64, 64, 3, 3)), "b3": rng.normal(0, 0.5, 64),
        "W4": rng.normal(0, 0.02, (512, 3136)), "b4": rng.normal(0, 0.5, 512),
        "W5": rng.normal(0, 0.1, (nA, 512)), "b5": rng.normal(0, 0.5, nA),
    }
    return {k: v.astype(np.float32).astype(np.float64) for k, v in p.items()}


@pytest.mark.parametrize("optimizer,ps_mode", [("rmsprop", "aggregate"), ("adagrad", "per_message")])
def test_round_closed_form_constant_activations(optimizer, ps_mode):
    nA, B, C = 6, 12, 400
    gamma, lr, rho, eps, ada_eps = 0.9, 2.5e-4, 0.95, 0.01, 1e-8
    cfg = O.Config(n_actions=nA, batch=B, capacity=C, gamma=gamma, lr=lr, rms_rho=rho, rms_eps=eps,
                   optimizer=optimizer, ada_eps=ada_eps, ps_mode=ps_mode,
                   outlier_enabled=False, target_period=1000)
    p = constant_activation_params(nA)
    theta0 = np.concatenate([p[n].ravel() for n, _ in O.param_shapes(nA)])
    orc = O.GorilaOracle(cfg, theta0)
    f = synth.frames(synth.SEED_DATA, 0, 0, C)
    a, r, d = synth.meta(synth.SEED_DATA, 0, 0, C, nA)
    d = d.copy()
    d[::5] = 1                              # make sure both TD branches occur
    orc.insert(0, f, a, r, d)
    info = orc.round(0)["learners"][0]
    assert info["accepted"]

    # forward: constant planes, R18 flatten order
    z1 = p["b1"]; a1 = np.maximum(z1, 0)
    z2 = p["W2"].sum(axis=(2, 3)) @ a1 + p["b2"]; a2 = np.maximum(z2, 0)
    z3 = p["W3"].sum(axis=(2, 3)) @ a2 + p["b3"]; a3 = np.maximum(z3, 0)
    x4 = np.repeat(a3, 49)
    z4 = p["W4"] @ x4 + p["b4"]; a4 = np.maximum(z4, 0)
    q = p["W5"] @ a4 + p["b5"]
    for z in (z1, z2, z3, z4):               # masks must be mixed and unambiguous
        assert (z > 0).any() and (z < 0).any() and np.abs(z).min() > 1e-6
    np.testing.assert_allclose(info["Q"], np.tile(q, (B, 1)), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(info["Qhat"], np.tile(q, (B, 1)), rtol=1e-12, atol=1e-12)

    # TD (Alg. 1): Q̂ = Q here since θ⁻ = θ at init
    ai, ri, di = np.asarray(info["a"], int), np.asarray(info["r"], np.float64), np.asarray(info["d"])
    assert di.any() and not di.all()
    y = ri + np.where(di != 0, 0.0, gamma * q.max())
    delta = y - q[ai]
    np.testing.assert_allclose(info["y"], y, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(info["delta"], delta, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(info["loss"], np.mean(delta ** 2), rtol=1e-12)
    dQ = np.zeros((B, nA))
    dQ[np.arange(B), ai] = -np.clip(delta, -1, 1) / B

    # backward, sample by sample (Eq. 2)
    s, _, _, _, _ = orc.learners[0].ring.gather(info["tau"])
    x = np.asarray(s, np.float64) / 255.0
    m1, m2, m3, m4 = (z1 > 0), (z2 > 0), (z3 > 0), (z4 > 0)
    G = {n: np.zeros(sh) for n, sh in O.param_shapes(nA)}
    for i in range(B):
        G["W5"] += np.outer(dQ[i], a4); G["b5"] += dQ[i]
        g4 = m4 * (p["W5"].T @ dQ[i])
        G["W4"] += np.outer(g4, x4); G["b4"] += g4
        g3 = m3[:, None, None] * (p["W4"].T @ g4).reshape(64, 7, 7)
        G["W3"] += g3.sum(axis=(1, 2))[:, None, None, None] * a2[None, :, None, None]
        G["b3"] += g3.sum(axis=(1, 2))
        g2 = m2[:, None, None] * _convT(p["W3"], g3, 1, 9)
        G["W2"] += g2.sum(axis=(1, 2))[:, None, None, None] * a1[None, :, None, None]
        G["b2"] += g2.sum(axis=(1, 2))
        g1 = m1[:, None, None] * _convT(p["W2"], g2, 2, 20)
        for kh in range(8):
            for kw in range(8):
                G["W1"][:, :, kh, kw] += np.einsum("ohw,chw->oc", g1, x[i][:, kh:kh + 77:4, kw:kw + 77:4])
        G["b1"] += g1.sum(axis=(1, 2))
    g = np.concatenate([G[n].ravel() for n, _ in O.param_shapes(nA)])
    for (n, _), lo in zip(O.param_shapes(nA), np.cumsum([0] + [G[n].size for n, _ in O.param_shapes(nA)])):
        got = info["G"][lo:lo + G[n].size]
        scale = max(np.abs(G[n]).max(), 1e-300)
        assert np.abs(G[n]).max() > 0, n
        np.testing.assert_allclose(got, G[n].ravel(), rtol=0, atol=1e-11 * scale, err_msg=n)

    if optimizer == "rmsprop":  # first centered-RMSProp step from m = v = 0 (reading R2), closed form
        theta1 = theta0 - lr * g / np.sqrt(rho * (1 - rho) * g * g + eps)
    else:  # first AdaGrad step from an empty accumulator: θ − η g / (|g| + ε)
        theta1 = theta0 - lr * g / (np.abs(g) + ada_eps)
    np.testing.assert_allclose(orc.theta, theta1, rtol=0, atol=1e-15)
    assert orc.V == 1
