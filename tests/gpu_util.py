"""Shared helpers of the -m gpu parity tests: build a GPU context and an oracle on the
same seeded inputs, teacher-force the oracle from the GPU state, and compare."""
import numpy as np

import oracle as O
import synth

TOL = {"fp32": {"q": 1e-5, "g": 1e-5, "dtheta": 1e-5, "loss": 1e-5, "g_kink": 5e-3},
       "bf16": {"q": 1e-3, "g": 5e-3, "dtheta": 5e-3, "loss": 1e-3, "g_kink": 2e-2}}


def make_pair(nA=4, B=32, C=2000, n_insert=2000, math="fp32", L=1, history=2, p_poison=0.0, terminals=None, **kw):
    from paper_1507_04296_b200 import Gorila
    theta0 = kw.pop("theta0", None)
    if theta0 is None:
        theta0 = synth.theta0(nA)
    g = Gorila(n_actions=nA, batch=B, replay_capacity=C, n_learners_local=L, theta0=theta0, math=math,
               history=history, **kw)
    ocfg = O.Config(n_actions=nA, batch=B, capacity=C, learners=tuple(range(L)),
                    mode="bf16" if math == "bf16" else "exact", gamma=kw.get("gamma", 0.99),
                    lr=kw.get("lr", 2.5e-4), rms_rho=kw.get("rms_rho", 0.95), rms_eps=kw.get("rms_eps", 0.01),
                    optimizer=kw.get("optimizer", "rmsprop"), ada_eps=kw.get("ada_eps", 1e-8),
                    target_period=kw.get("target_period", 100), max_staleness=kw.get("max_staleness", -1),
                    outlier_enabled=bool(kw.get("outlier_enabled", True)), outlier_warmup=kw.get("outlier_warmup", 100),
                    outlier_k=kw.get("outlier_k", 3.0), outlier_beta=kw.get("outlier_beta", 0.999),
                    min_replay=kw.get("min_replay", 1), seed_sample=kw.get("seed", 1507),
                    ps_mode=kw.get("ps_mode", "aggregate"), replay_mode=kw.get("replay_mode", "local"))
    orc = O.GorilaOracle(ocfg, theta0)
    for j in range(L):
        f = synth.frames(synth.SEED_DATA, j, 0, n_insert)
        a, r, d = synth.meta(synth.SEED_DATA, j, 0, n_insert, nA, p_poison)
        if terminals is not None:
            d = terminals(j, d)
        g.replay_insert(j, f, a, r, d)
        orc.insert(j, f, a, r, d)
    return g, orc


def teacher_force(g, orc):
    """Copy the GPU's PS and learner state into the oracle (one-step parity)."""
    th, m, v, V = g.get_state()
    orc.theta = th.astype(np.float64)
    orc.m = m.astype(np.float64)
    orc.v = v.astype(np.float64)
    orc.V = int(V)
    for j, L in orc.learners.items():
        tm, st = g.get_learner_state(j)
        L.theta_minus = tm.astype(np.float64)
        L.stats = O.LossStats(mu=st["mu"], var=st["var"], count=st["count"])
        L.last_sync = st["last_sync"]
    orc.history = {}


def rel_inf(x, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(np.asarray(x, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


def rel_l2(x, ref):
    ref = np.asarray(ref, np.float64)
    nr = np.linalg.norm(ref)
    if nr == 0:
        return 0.0 if np.linalg.norm(x) == 0 else np.inf
    return float(np.linalg.norm(np.asarray(x, np.float64) - ref) / nr)


def per_tensor_rel_l2(x, ref, nA):
    out, off = {}, 0
    for name, shp in O.param_shapes(nA):
        n = int(np.prod(shp))
        out[name] = rel_l2(x[off:off + n], ref[off:off + n])
        off += n
    return out


def run_round_both(g, orc, k, learners, staleness=None):
    """One round on both sides. Returns (gpu dict, oracle dict)."""
    stal = None if staleness is None else [staleness.get(j, 0) for j in learners]
    th0 = g.get_state()[0]
    info = g.learner_step(learners, k, staleness=stal)
    G = g.get_grad()
    qs = {j: g.get_q(j) for j in learners}
    ri = g.ps_apply_shard(k)
    synced = g.sync_target(learners)
    th1, m1, v1, V1 = g.get_state()
    gpu = {"info": dict(zip(learners, info)), "G": G, "q": qs, "round": ri, "synced": dict(zip(learners, synced)),
           "theta0": th0, "theta1": th1, "V": V1}
    res = orc.round(k, staleness=staleness)
    return gpu, res


def mask_flip_layer(g, acts, max_frac=1e-4, rel=1e-3):
    """Observed kink rule (R30): the deepest conv / fc4 layer whose ReLU mask differs between
    the GPU's saved activations of its last learner step (gorila_get_activation) and the oracle's (acts
    of O.qnet_forward on the same batch), 0 if none. Only ambiguous decisions qualify: at most max_frac
    of the layer's elements, every one with both values within rel * max|a| of zero; anything else is a
    real discrepancy and fails here."""
    B = acts.shape[0]
    sizes = [("a1", (20, 20, 32)), ("a2", (9, 9, 64)), ("a3", (7, 7, 64)), ("a4", (512,))]
    off, deepest = 0, 0
    for l, (name, shp) in enumerate(sizes, start=1):
        n = int(np.prod(shp))
        ref = acts[:, off:off + n]
        off += n
        got = g.get_activation(name).reshape(B, -1)
        if len(shp) == 3:  # GPU NHWC -> oracle CHW
            got = got.reshape((B,) + shp).transpose(0, 3, 1, 2).reshape(B, -1)
        flips = (got > 0) != (ref > 0)
        nf = int(flips.sum())
        if nf == 0:
            continue
        big = max(float(np.abs(ref).max()), 1e-30)
        assert nf <= max(1, max_frac * ref.size), (name, "mask flips", nf, ref.size)
        assert np.all(np.abs(got[flips]) <= rel * big) and np.all(np.abs(ref[flips]) <= rel * big), \
            (name, "flipped elements not near zero", float(np.abs(got[flips]).max()), float(np.abs(ref[flips]).max()), big)
        deepest = l
    return deepest


def round_bf16_vec(t):
    """Vectorised oracle/oracle.c::orc_round_bf16 (frexp, 8 significant bits, ties to even)."""
    m, e = np.frexp(np.asarray(t, np.float64))
    return np.ldexp(np.rint(np.ldexp(m, 8)), e - 8)


def replica_of(theta, nA, math):
    """theta^- as the replica holds it: conv / fc4 weights bf16 in bf16 mode, the rest fp32 (R16)."""
    out = np.asarray(theta, np.float64).copy()
    if math != "bf16":
        return out
    off = 0
    for name, shp in O.param_shapes(nA):
        n = int(np.prod(shp))
        if name in ("W1", "W2", "W3", "W4"):
            out[off:off + n] = round_bf16_vec(out[off:off + n])
        off += n
    return out


LAYER_OF = {"W1": 1, "b1": 1, "W2": 2, "b2": 2, "W3": 3, "b3": 3, "W4": 4, "b4": 4, "W5": 5, "b5": 5}


def ambiguous_layer(theta, s, nA, rel=1e-6, mode="exact"):
    """Kink rule (R30): the deepest hidden layer l (1..4) with a pre-activation |z| <= rel * max|z|,
    recomputed with the oracle's layer primitives at the oracle's rounding points for `mode`; 0 if none.
    A ReLU decision that close to 0 is decided differently by fp32 accumulation (and, in bf16 mode, by a
    one-ulp difference of a rounded input activation), which moves the gradients of tensors at and below
    layer l."""
    p = O.unflatten(np.asarray(theta, np.float64), nA)
    bf = mode == "bf16"

    def q(t):
        return round_bf16_vec(t) if bf else t

    if bf:  # oracle BF16 mode: bf16 weights and a1..a3, raw bytes into conv1, 1/255 (fp32) on its sum
        z1 = O.conv2d_fwd(s.astype(np.float64), q(p["W1"]), None, 4) * float(np.float32(1.0) / np.float32(255.0))
        z1 = z1 + p["b1"][None, :, None, None]
    else:
        z1 = O.conv2d_fwd(s.astype(np.float64) / 255.0, p["W1"], p["b1"], 4)
    z2 = O.conv2d_fwd(q(np.maximum(z1, 0)), q(p["W2"]), p["b2"], 2)
    z3 = O.conv2d_fwd(q(np.maximum(z2, 0)), q(p["W3"]), p["b3"], 1)
    z4 = O.linear_fwd(q(np.maximum(z3, 0)).reshape(len(s), -1), q(p["W4"]), p["b4"])
    deepest = 0
    for l, z in enumerate((z1, z2, z3, z4), start=1):
        if np.any(np.abs(z) <= rel * np.max(np.abs(z))):
            deepest = l
    return deepest
