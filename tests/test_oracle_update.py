"""Pins for the oracle's TD / discard / PS-update logic and for the round as a whole.

References: SPEC/hand worked examples (tests/golden/), closed forms, an
exponentially-weighted-moment closed form, torch autograd (Huber loss), and
invariants BASELINE.json names (no update when rewards and Q agree; target
net immutable between syncs).
"""
import json
import os

import numpy as np
import torch

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_td_target_and_loss_worked_examples():
    g = _gold("td_cases.json")
    for c in g["target"]:
        nA = 3
        Qhat = np.full((1, nA), -50.0)
        Qhat[0, 1] = c["max_qhat"]
        y, _, _, _, _ = O.td_terms(np.zeros((1, nA)), Qhat, [0], [c["r"]], [c["terminal"]], c["gamma"])
        assert abs(y[0] - c["y"]) < 1e-12, c
    for c in g["loss"]:
        Q = np.array([[c["q"], 0.0]])
        # terminal with r = y pins y exactly
        _, delta, dQ, loss, ell = O.td_terms(Q, np.zeros((1, 2)), [0], [c["y"]], [1], 0.99)
        assert abs(loss - c["loss"]) < 1e-12 and abs(delta[0] - c["delta"]) < 1e-12
        assert abs(ell - abs(c["delta"])) < 1e-12


def test_td_invariants():
    rng = np.random.default_rng(0)
    B, nA = 64, 6
    Q, Qhat = rng.standard_normal((B, nA)), rng.standard_normal((B, nA))
    a = rng.integers(0, nA, B)
    r = rng.choice([-1.0, 0.0, 1.0], B)
    d = rng.integers(0, 2, B)
    # gamma = 1 with a zero target net -> y = r
    y, _, _, _, _ = O.td_terms(Q, np.zeros_like(Qhat), a, r, np.zeros(B), 1.0)
    assert (y == r).all()
    y, delta, dQ, loss, ell = O.td_terms(Q, Qhat, a, r, d, 0.99)
    assert loss >= 0 and ell >= 0
    # only the taken action's column carries gradient; clip bounds it by 1/B
    mask = np.zeros_like(dQ, bool)
    mask[np.arange(B), a] = True
    assert (dQ[~mask] == 0).all() and np.abs(dQ).max() <= 1.0 / B


def test_clipped_error_is_huber_gradient():
    # R3: clipping delta in Eq.2 == gradient of the Huber(1) loss, mean over the batch
    rng = np.random.default_rng(1)
    B, nA = 40, 5
    Q = rng.standard_normal((B, nA)) * 3
    Qhat = rng.standard_normal((B, nA)) * 3
    a = rng.integers(0, nA, B)
    r = rng.choice([-1.0, 0.0, 1.0], B)
    d = rng.integers(0, 2, B)
    y, delta, dQ, _, _ = O.td_terms(Q, Qhat, a, r, d, 0.9)
    assert (np.abs(delta) > 1).any() and (np.abs(delta) < 1).any()
    Qt = torch.from_numpy(Q).requires_grad_()
    qa = Qt[torch.arange(B), torch.from_numpy(a)]
    torch.nn.functional.huber_loss(qa, torch.from_numpy(y), delta=1.0, reduction="mean").backward()
    assert np.allclose(dQ, Qt.grad.numpy(), rtol=0, atol=1e-15)
    # |delta| <= 1 reproduces Eq.2's unclipped (y - Q) factor exactly
    small = np.abs(delta) <= 1
    assert np.allclose(dQ[np.arange(B), a][small], -delta[small] / B, rtol=0, atol=0)


def test_staleness_and_sync_worked_examples():
    g = _gold("ps_cases.json")
    for c in g["staleness"]:
        assert O.is_stale(c["current"], c["base"], c["max_delay"]) == c["stale"]
    for c in g["sync"]:
        assert O.should_sync(c["version"], c["last"], c["period"]) == c["sync"]
        if "last_after" in c:  # single-shot catch-up: 0 -> 12 syncs once, last = 12
            assert not O.should_sync(c["then_version"], c["last_after"], c["period"])


def test_outlier_worked_example_and_warmup():
    for c in _gold("ps_cases.json")["outlier"]:
        st = O.LossStats(mu=c["mu"], var=c["sigma"] ** 2, count=1000)
        assert st.rejects(c["loss"], c["k"], warmup=100) == c["rejected"]
        st.count = 5  # before warm-up nothing is rejected
        assert not st.rejects(1e9, c["k"], warmup=100)


def test_loss_stats_ema_closed_form():
    # EMA recurrence == exponentially weighted mean / variance with explicit weights
    # w_1 = beta^(n-1), w_i = (1-beta) beta^(n-i): sum w = 1, var = sum w (x - mu_n)^2
    rng = np.random.default_rng(2)
    x = rng.standard_normal(300) * 0.3 + 1.0
    beta = 0.99
    st = O.LossStats()
    st.update(x[0], beta)
    assert st.mu == x[0] and st.var == 0.0  # first observation
    for v in x[1:]:
        st.update(v, beta)
    n = len(x)
    w = np.array([beta ** (n - 1)] + [(1 - beta) * beta ** (n - i) for i in range(2, n + 1)])
    mu = (w * x).sum()
    var = (w * (x - mu) ** 2).sum()
    assert abs(st.mu - mu) < 1e-12 and abs(st.var - var) < 1e-12
    c = O.LossStats()
    for _ in range(2000):
        c.update(0.7, beta)
    assert abs(c.mu - 0.7) < 1e-12 and c.var < 1e-20  # constant stream


def test_rmsprop_closed_forms():
    g = _gold("ps_cases.json")["rmsprop_first_step"]
    th, m, v = np.array([0.0]), np.array([0.0]), np.array([0.0])
    O.rmsprop_apply(th, m, v, np.array([g["g"]]), g["lr"], g["rho"], g["eps"])
    assert abs(m[0] - g["m"]) < 1e-15 and abs(v[0] - g["v"]) < 1e-15
    assert abs(th[0] - g["delta_theta"]) < 1e-12
    # zero gradient: theta unchanged bitwise (m, v decay)
    th, m, v = np.array([0.3]), np.array([0.1]), np.array([0.2])
    O.rmsprop_apply(th, m, v, np.array([0.0]), 1e-3, 0.95, 0.01)
    assert th[0] == 0.3 and abs(m[0] - 0.095) < 1e-15
    # constant g for T steps: m_T = (1 - rho^T) g, v_T = (1 - rho^T) g^2
    th, m, v = np.zeros(1), np.zeros(1), np.zeros(1)
    for _ in range(37):
        O.rmsprop_apply(th, m, v, np.array([-2.0]), 1e-3, 0.9, 0.01)
    assert abs(m[0] - (1 - 0.9 ** 37) * -2.0) < 1e-13 and abs(v[0] - (1 - 0.9 ** 37) * 4.0) < 1e-13


def test_adagrad_worked_example():
    g = _gold("ps_cases.json")["adagrad_first_step"]
    th, acc = np.array([g["theta"]]), np.array([0.0])
    O.adagrad_apply(th, acc, np.array([g["g"]]), g["lr"], g["eps"])
    assert acc[0] == g["acc"] and abs(th[0] - g["theta_after"]) < 1e-12
    d1 = g["theta"] - th[0]
    prev = th[0]
    O.adagrad_apply(th, acc, np.array([g["g"]]), g["lr"], g["eps"])
    assert prev - th[0] < d1  # second identical step is smaller


def test_shard_bounds_disjoint_cover():
    P = O.param_count(18)
    for W in (1, 2, 4, 8, 31):
        b = O.shard_bounds(P, W)
        assert b[0][0] == 0 and b[-1][1] == P and len(b) == W
        assert all(b[i][1] == b[i + 1][0] for i in range(W - 1))


# ------------------------------------------------------------------ whole rounds

def _filled_oracle(cfg, n_frames, learner_ids=(0,), p_poison=0.0):
    orc = O.GorilaOracle(cfg, synth.theta0(cfg.n_actions))
    for j in learner_ids:
        f = synth.frames(synth.SEED_DATA, j, 0, n_frames)
        a, r, d = synth.meta(synth.SEED_DATA, j, 0, n_frames, cfg.n_actions, p_poison)
        orc.insert(j, f, a, r, d)
    return orc


def test_round_shard_count_invariance():
    res = []
    for W in (1, 2, 4, 8, 31):
        cfg = O.Config(n_actions=4, batch=8, capacity=600, n_shards=W)
        orc = _filled_oracle(cfg, 600)
        orc.round(0)
        orc.round(1)
        res.append(orc.theta.copy())
    for t in res[1:]:
        assert (t == res[0]).all()


def test_no_update_invariant():
    # zero weights, fc5 bias = 1, gamma = 0.75: r = 0.25 (non-terminal) or 1.0 (terminal)
    # -> y == Q == 1 exactly -> delta == 0 -> G == 0 -> theta bitwise unchanged (BASELINE.json)
    nA = 4
    cfg = O.Config(n_actions=nA, batch=16, capacity=300, gamma=0.75, outlier_enabled=False)
    theta0 = np.zeros(O.param_count(nA), np.float32)
    theta0[-nA:] = 1.0
    orc = O.GorilaOracle(cfg, theta0)
    f = synth.frames(synth.SEED_DATA, 0, 0, 300)
    a, _, d = synth.meta(synth.SEED_DATA, 0, 0, 300, nA)
    d = d.copy()
    d[::7] = 1
    r = np.where(d == 1, 1.0, 0.25).astype(np.float32)
    orc.insert(0, f, a, r, d)
    before = orc.theta.copy()
    for k in range(3):
        info = orc.round(k)
        L = info["learners"][0]
        assert (L["delta"] == 0).all() and L["loss"] == 0.0 and (L["G"] == 0).all()
    assert (orc.theta == before).all() and orc.V == 3


def test_target_net_immutable_between_syncs_and_synced_at_period():
    cfg = O.Config(n_actions=4, batch=8, capacity=500, target_period=3, outlier_enabled=False)
    orc = _filled_oracle(cfg, 500)
    tm0 = orc.learners[0].theta_minus.copy()
    assert (tm0 == orc.theta).all()  # theta^- = theta at init (Alg.1)
    synced_rounds = []
    for k in range(7):
        before = orc.learners[0].theta_minus.copy()
        info = orc.round(k)
        if info["synced"][0]:
            synced_rounds.append(k)
            assert (orc.learners[0].theta_minus == orc.theta).all()
        else:
            assert (orc.learners[0].theta_minus == before).all()
    assert synced_rounds == [2, 5]  # V = 3 after round 2, 6 after round 5


def test_poison_reward_is_rejected_and_leaves_theta_unchanged():
    # reward 1e6 -> rejected_outlier, no parameter change
    nA = 4
    cfg = O.Config(n_actions=nA, batch=8, capacity=400, outlier_warmup=3)
    orc = _filled_oracle(cfg, 400)
    for k in range(4):
        orc.round(k)
    ring = orc.learners[0].ring
    ring.r[:] = 1e6
    ring.d[:] = 1
    th, V = orc.theta.copy(), orc.V
    info = orc.round(4)
    L = info["learners"][0]
    assert L["rejected_outlier"] and not L["accepted"] and info["n_accepted"] == 0
    assert (orc.theta == th).all() and orc.V == V


def test_stale_gradients_discarded_with_scheduled_delay():
    nA = 4
    cfg = O.Config(n_actions=nA, batch=8, capacity=400, learners=(0, 1, 2), max_staleness=4,
                   outlier_enabled=False)
    orc = _filled_oracle(cfg, 400, learner_ids=(0, 1, 2))
    for k in range(3):
        orc.round(k)  # V = 9
    info = orc.round(3, staleness={1: 2})  # learner 1 computes on theta^(1): b = V^(1) = 3, V0 = 9 -> stale
    assert info["learners"][1]["stale"] and not info["learners"][1]["accepted"]
    assert info["learners"][1]["base_version"] == 3
    assert info["n_accepted"] == 2 and info["version_after"] == 11
    info = orc.round(4, staleness={2: 1})  # b = V^(3) = 9, V0 = 11 -> delay 2 <= 4 accepted
    assert not info["learners"][2]["stale"] and info["n_accepted"] == 3


def test_serial_equivalence_with_torch_autograd_loop():
    """one learner, staleness off, rejection off == a plain serial DQN loop.

    The loop below uses torch autograd + the Huber(1) loss for the gradient and
    the centered-RMSProp definition (R2) for the update.
    """
    nA, B, C = 4, 8, 300
    cfg = O.Config(n_actions=nA, batch=B, capacity=C, outlier_enabled=False, target_period=2)
    orc = _filled_oracle(cfg, C)
    theta = torch.from_numpy(synth.theta0(nA).astype(np.float64))
    theta_minus = theta.clone()
    m, v = torch.zeros_like(theta), torch.zeros_like(theta)
    shapes = O.param_shapes(nA)

    def net(th, x):
        p, off = {}, 0
        for name, shp in shapes:
            n = int(np.prod(shp))
            p[name] = th[off:off + n].reshape(shp)
            off += n
        h = torch.relu(torch.nn.functional.conv2d(x / 255.0, p["W1"], p["b1"], stride=4))
        h = torch.relu(torch.nn.functional.conv2d(h, p["W2"], p["b2"], stride=2))
        h = torch.relu(torch.nn.functional.conv2d(h, p["W3"], p["b3"], stride=1))
        h = torch.relu(torch.nn.functional.linear(h.reshape(h.shape[0], -1), p["W4"], p["b4"]))
        return torch.nn.functional.linear(h, p["W5"], p["b5"])

    ring = orc.learners[0].ring
    for k in range(4):
        tau = O.sample_indices(ring.n, ring.size, B, cfg.seed_sample, 0, k)
        s, s2, a, r, d = ring.gather(tau)
        with torch.no_grad():
            qn = net(theta_minus, torch.from_numpy(s2.astype(np.float64))).max(1).values
        y = torch.from_numpy(r.astype(np.float64)) + cfg.gamma * qn * torch.from_numpy(1.0 - d)
        th = theta.clone().requires_grad_()
        q = net(th, torch.from_numpy(s.astype(np.float64)))[torch.arange(B), torch.from_numpy(a.astype(np.int64))]
        torch.nn.functional.huber_loss(q, y, delta=1.0, reduction="mean").backward()
        g = th.grad
        m = cfg.rms_rho * m + (1 - cfg.rms_rho) * g
        v = cfg.rms_rho * v + (1 - cfg.rms_rho) * g * g
        theta = theta - cfg.lr * g / torch.sqrt(v - m * m + cfg.rms_eps)
        if (k + 1) % 2 == 0:
            theta_minus = theta.clone()
        orc.round(k)
        assert np.allclose(orc.theta, theta.numpy(), rtol=0, atol=1e-13)
    assert np.allclose(orc.learners[0].theta_minus, theta_minus.numpy(), rtol=0, atol=1e-13)


def test_descent_on_frozen_batch():
    # repeated steps on a fixed batch with the target frozen decrease the loss
    nA, B = 4, 8
    theta = synth.theta0(nA).astype(np.float64)
    rng = np.random.default_rng(9)
    s = rng.integers(0, 256, size=(B, 4, 84, 84), dtype=np.uint8)
    a = rng.integers(0, nA, B)
    y = rng.standard_normal(B) * 0.3
    m, v = np.zeros_like(theta), np.zeros_like(theta)
    losses = []
    for _ in range(5):
        Q, acts = O.qnet_forward(theta, s, nA)
        _, delta, dQ, loss, _ = O.td_terms(Q, np.zeros((B, nA)), a, y, np.ones(B), 0.0)
        losses.append(loss)
        O.rmsprop_apply(theta, m, v, O.qnet_backward(theta, s, acts, dQ, nA), 2.5e-4, 0.95, 0.01)
    assert all(l1 < l0 for l0, l1 in zip(losses, losses[1:]))


# ---------------------------------------------------------------- NEXT row f1: per-message PS (R32)
def _f1_pair(ps_mode, learners, optimizer="adagrad", rounds=2):
    nA, B, C = 4, 8, 400
    cfg = O.Config(n_actions=nA, batch=B, capacity=C, learners=learners, outlier_warmup=1,
                   optimizer=optimizer, lr=1e-3, ps_mode=ps_mode)
    orc = O.GorilaOracle(cfg, synth.theta0(nA))
    for j in learners:
        f = synth.frames(synth.SEED_DATA, j, 0, C)
        a, r, d = synth.meta(synth.SEED_DATA, j, 0, C, nA)
        orc.insert(j, f, a, r, d)
    return orc


def test_f1_single_message_equals_aggregate():
    """One accepted message per round: a step on it == a step on the mean of one (bitwise)."""
    for opt in ("adagrad", "rmsprop"):
        a, b = _f1_pair("aggregate", (0,), opt), _f1_pair("per_message", (0,), opt)
        for k in range(3):
            a.round(k)
            b.round(k)
        assert np.array_equal(a.theta, b.theta) and np.array_equal(a.v, b.v) and a.V == b.V


def test_f1_messages_applied_one_step_each_in_learner_order():
    """Two learners: theta moves by the optimizer applied to G_0 then G_1 (the PS
    applies each learner's gradient as its own update), V += 1 per message, and it differs from
    one step on the mean (the optimizer is nonlinear in its state)."""
    for opt in ("adagrad", "rmsprop"):
        orc = _f1_pair("per_message", (0, 1), opt)
        agg = _f1_pair("aggregate", (0, 1), opt)
        th0, m0, v0 = orc.theta.copy(), orc.m.copy(), orc.v.copy()
        res = orc.round(0)
        agg.round(0)
        G0, G1 = res["learners"][0]["G"], res["learners"][1]["G"]
        assert res["learners"][0]["accepted"] and res["learners"][1]["accepted"]
        th, m, v = th0.copy(), m0.copy(), v0.copy()
        for G in (G0, G1):  # the pinned primitives, composed in ascending learner id
            if opt == "adagrad":
                O.adagrad_apply(th, v, G, 1e-3, 1e-8)
            else:
                O.rmsprop_apply(th, m, v, G, 1e-3, 0.95, 0.01)
        assert np.array_equal(orc.theta, th) and orc.V == 2 and res["n_accepted"] == 2
        assert not np.allclose(orc.theta, agg.theta, rtol=0, atol=1e-12)


def _f1_pair_cfg(learners, **kw):
    nA, B, C = 4, 8, 400
    cfg = O.Config(n_actions=nA, batch=B, capacity=C, learners=learners, outlier_warmup=1, outlier_enabled=False,
                   optimizer="adagrad", lr=1e-3, ps_mode="per_message", **kw)
    orc = O.GorilaOracle(cfg, synth.theta0(nA))
    for j in learners:
        f = synth.frames(synth.SEED_DATA, j, 0, C)
        a, r, d = synth.meta(synth.SEED_DATA, j, 0, C, nA)
        orc.insert(j, f, a, r, d)
    return orc


def test_f1_staleness_judged_against_the_version_at_arrival():
    """Hand case ("discards gradients older than a threshold"; P:160 V counts PS updates):
    max delay 1, three messages computed on the replica of version V0. Message 1 arrives at V0 (delay
    0: applied, V = V0 + 1), message 2 at V0 + 1 (delay 1: applied, V = V0 + 2), message 3 at V0 + 2
    (delay 2 > 1: discarded). Judged against V0 alone (round-start reading) all three would pass."""
    orc = _f1_pair_cfg((0, 1, 2), max_staleness=1)
    th0, v0 = orc.theta.copy(), orc.v.copy()
    res = orc.round(0)
    L = res["learners"]
    assert [L[j]["base_version"] for j in (0, 1, 2)] == [0, 0, 0]
    assert [L[j]["version_at_arrival"] for j in (0, 1, 2)] == [0, 1, 2]
    assert [bool(L[j]["accepted"]) for j in (0, 1, 2)] == [True, True, False]
    assert [bool(L[j]["stale"]) for j in (0, 1, 2)] == [False, False, True]
    assert res["n_accepted"] == 2 and orc.V == 2
    th, v = th0.copy(), v0.copy()
    for j in (0, 1):  # the pinned AdaGrad primitive, the two fresh messages in learner order
        O.adagrad_apply(th, v, L[j]["G"], 1e-3, 1e-8)
    assert np.array_equal(orc.theta, th) and np.array_equal(orc.v, v)
    # next round: both delays restart from the new replica (base V = 2)
    res = orc.round(1)
    assert [res["learners"][j]["base_version"] for j in (0, 1, 2)] == [2, 2, 2]
    assert [bool(res["learners"][j]["accepted"]) for j in (0, 1, 2)] == [True, True, False]


def test_f1_target_sync_at_the_first_version_inside_the_round():
    """N = 2, three fresh messages from V = 0 (theta^- = theta^+ "after every N gradient
    updates in the central parameter server"): the sync fires after message 2 (V = 2 >= 0 + 2), so
    theta^- is theta after two steps and last = 2; message 3 (V = 3 < 4) does not sync again. A
    round-end reading would copy theta after three steps with last = 3."""
    orc = _f1_pair_cfg((0, 1, 2), target_period=2)
    th0, v0 = orc.theta.copy(), orc.v.copy()
    res = orc.round(0)
    L = res["learners"]
    th, v = th0.copy(), v0.copy()
    O.adagrad_apply(th, v, L[0]["G"], 1e-3, 1e-8)
    O.adagrad_apply(th, v, L[1]["G"], 1e-3, 1e-8)
    th2 = th.copy()
    O.adagrad_apply(th, v, L[2]["G"], 1e-3, 1e-8)
    assert np.array_equal(orc.theta, th) and orc.V == 3
    for j in (0, 1, 2):
        assert res["synced"][j]
        assert np.array_equal(orc.learners[j].theta_minus, th2)
        assert orc.learners[j].last_sync == 2
    assert not np.array_equal(th2, th)
    # N = 1: every step syncs; theta^- ends at the round's last version
    orc = _f1_pair_cfg((0, 1, 2), target_period=1)
    orc.round(0)
    assert all(np.array_equal(orc.learners[j].theta_minus, orc.theta) and orc.learners[j].last_sync == 3
               for j in (0, 1, 2))
