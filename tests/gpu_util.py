"""Shared helpers of the -m gpu parity tests: build a GPU context and an oracle on the
same seeded inputs, teacher-force the oracle from the GPU state, and compare."""
import numpy as np

import oracle as O
import synth

TOL = {"fp32": {"q": 1e-5, "g": 1e-5, "dtheta": 1e-5, "loss": 1e-5},
       "bf16": {"q": 1e-3, "g": 5e-3, "dtheta": 5e-3, "loss": 1e-3}}

# DESIGN.md R30 (teacher-forced ReLU decisions). A ReLU whose pre-activation lies within accumulation
# error of 0 is decided by rounding order (fp32 vs fp64 sums; in bf16 mode also by a one-ulp different
# rounding of an input activation), and its decision switches a whole gradient path on or off. Where
# the GPU and the oracle decide such an element differently, the oracle's backward takes the GPU's
# activation value for that element (its mask bit and its wgrad input) -- only there: the oracle's
# pre-activation and the GPU's value must both lie within BAND * max|z_l| of 0, and at most
# FORCED_MAX_FRAC of the layer may be forced. Every gradient and update is then compared at the full
# tolerance above.
BAND = {"fp32": 1e-4, "bf16": 2e-3}
FORCED_MAX_FRAC = 1e-4
ACT_LAYERS = (("a1", (20, 20, 32)), ("a2", (9, 9, 64)), ("a3", (7, 7, 64)), ("a4", (512,)))


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
                    ps_mode=kw.get("ps_mode", "aggregate") if kw.get("ps_mode") != "async" else "per_message",
                    replay_mode=kw.get("replay_mode", "local"))
    orc = O.GorilaOracle(ocfg, theta0)
    for j in range(L):
        f = synth.frames(synth.SEED_DATA, j, 0, n_insert)
        a, r, d = synth.meta(synth.SEED_DATA, j, 0, n_insert, nA, p_poison)
        if terminals is not None:
            d = terminals(j, d)
        g.replay_insert(j, f, a, r, d)
        orc.insert(j, f, a, r, d)
    return g, orc


def gpu_acts(g, learner=None, rows=None):
    """The GPU's a1..a4 of its last learner step in the oracle's layout ([B][a1|a2|a3|a4], CHW per
    sample, float64): learner None = the shared scratch (the last learner that ran), else learner's
    captured copy (Gorila.capture_activations). rows: only these samples."""
    parts = []
    for name, shp in ACT_LAYERS:
        x = g.get_activation(name) if learner is None else g.get_learner_activation(learner, name)
        x = x.reshape((g.batch,) + shp)
        if rows is not None:
            x = x[rows]
        if len(shp) == 3:  # NHWC -> CHW
            x = x.transpose(0, 3, 1, 2)
        parts.append(x.reshape(x.shape[0], -1))
    return np.concatenate(parts, axis=1).astype(np.float64)


def teacher_forced_acts(gpu, acts, zs, math, log=None):
    """R30: the oracle's activations `acts` (pre-activations `zs`) with the GPU's value `gpu` taken at
    every element whose ReLU decision differs -- asserting that each such decision is ambiguous (both
    |z_oracle| and |a_gpu| within BAND * max|z_l|) and that they are few (<= FORCED_MAX_FRAC of the
    layer). Any other difference is a real discrepancy and fails here. log (list) receives the number
    of forced elements per layer."""
    out = np.array(acts, np.float64, copy=True)
    off, forced = 0, {}
    for name, shp in ACT_LAYERS:
        n = int(np.prod(shp))
        sl = slice(off, off + n)
        off += n
        ref, got, z = acts[:, sl], gpu[:, sl], zs[:, sl]
        flips = (got > 0) != (ref > 0)
        nf = int(flips.sum())
        forced[name] = nf
        if nf == 0:
            continue
        band = BAND[math] * float(np.abs(z).max())
        assert nf <= max(2, FORCED_MAX_FRAC * ref.size), (name, "ReLU decisions differ at", nf, "of", ref.size)
        assert float(np.abs(z[flips]).max()) <= band and float(np.abs(got[flips]).max()) <= band, \
            (name, "differing ReLU decision outside the ambiguity band", float(np.abs(z[flips]).max()),
             float(np.abs(got[flips]).max()), band)
        blk = out[:, sl]
        blk[flips] = got[flips]
    if log is not None:
        log.append(forced)
    return out


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
    """One round on both sides (gorila_round: learner_step + ps_apply_shard + sync_target; the learner
    records are read after the round, when the per-message mode's PS-side decisions are final); the
    oracle's backward is teacher-forced to the GPU's ambiguous ReLU decisions (R30). The gradient
    buffers, Q and the captured activations are intact after the round (the apply only reads them).
    Returns (gpu dict, oracle dict)."""
    stal = None if staleness is None else np.array([staleness.get(j, 0) for j in learners], np.int32)
    th0 = g.get_state()[0]
    g.capture_activations(True)
    info, ri, synced = g.round(np.array(learners, np.int32), k, stal, want_info=True)
    G = g.get_grad()
    qs = {j: g.get_q(j) for j in learners}
    info_by = dict(zip(learners, info))
    acts = {j: gpu_acts(g, j) for j in learners if not info_by[j]["not_ready"]}
    th1, m1, v1, V1 = g.get_state()
    forced = []
    gpu = {"info": info_by, "G": G, "q": qs, "round": ri, "synced": dict(zip(learners, synced)),
           "theta0": th0, "theta1": th1, "V": V1, "forced": forced}
    res = orc.round(k, staleness=staleness,
                    acts_hook=lambda j, a, z: teacher_forced_acts(acts[j], a, z, g.math, forced))
    return gpu, res


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
