"""Gorila DQN learner update — plain CPU oracle (TEST INFRASTRUCTURE ONLY; see __init__).

Follows Algorithm 1's learner half and the parameter
server step by step, in the order SURVEY §8(c) O1-O12 and
DESIGN.md list. Heavy loops (conv/FC, Philox, stacking) are the direct
definitions in ``oracle.c``; everything else is written out here in numpy fp64.

Readings of the paper (R-numbers, DESIGN.md §"Readings"):
  R1/R2  RMSProp (centered, lr 2.5e-4, rho 0.95, eps 0.01 inside the sqrt) is
         the graded optimizer; the paper's AdaGrad is available too.
  R3/R4  the TD error multiplying grad Q is clipped to [-1,1]; the batch
         gradient is G = -(1/B) sum_i clip(delta_i) grad Q(s_i,a_i); theta -= step.
  R6/R7  reported loss = mean delta^2 (Eq.1); outlier statistic l = mean |delta|.
  R8     outlier filter: EMA (beta) mean/var of l, decide on pre-update stats,
         then update with every batch; warm-up count.
  R10    stale iff V0 - b > max_delay (global-version units; equality accepted).
  R12    one PS step per round on the mean of accepted gradients; V += |Acc|.
  R13    target sync iff V >= last + N, then last = V (single-shot catch-up).
  R14/15 frame ring; tau in [n-size, n-2]; zero-pad across episode / eviction.
"""
import ctypes
import dataclasses
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")

EXACT = 0
BF16 = 2
MODES = {"exact": EXACT, "fp32": EXACT, "bf16": BF16}

FRAME = 84 * 84
STACK = 4 * FRAME


def build(force=False):
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(SO) or os.path.getmtime(src) > os.path.getmtime(SO):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC",
                               "-fvisibility=hidden", "-o", SO, src, "-lm"])


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(SO)
        P = ctypes.c_void_p
        i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        L.orc_philox.argtypes = [P, P, P]
        L.orc_sample_indices.argtypes = [i64, i64, i32, u64, i32, u64, P]
        L.orc_sample_indices.restype = ctypes.c_int
        L.orc_sample_indices_global.argtypes = [i32, P, i64, i32, u64, i32, u64, P, P]
        L.orc_sample_indices_global.restype = ctypes.c_int
        L.orc_stack.argtypes = [i64, i64, P, P, i64, P]
        L.orc_gather.argtypes = [i64, i64, P, P, P, P, i32, P, P, P, P, P, P]
        for f in ("orc_conv2d_fwd", "orc_conv2d_bwd_data", "orc_conv2d_bwd_weight"):
            getattr(L, f).argtypes = [ctypes.c_int] * 7 + [P] * (4 if f != "orc_conv2d_bwd_data" else 3)
        L.orc_linear_fwd.argtypes = [ctypes.c_int] * 3 + [P] * 4
        L.orc_linear_bwd_data.argtypes = [ctypes.c_int] * 3 + [P] * 3
        L.orc_linear_bwd_weight.argtypes = [ctypes.c_int] * 3 + [P] * 4
        L.orc_round_bf16.argtypes = [ctypes.c_double]
        L.orc_round_bf16.restype = ctypes.c_double
        L.orc_param_count.argtypes = [ctypes.c_int]
        L.orc_param_count.restype = i64
        L.orc_acts_per_sample.restype = i64
        L.orc_qnet_forward.argtypes = [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P, P, P]
        L.orc_qnet_backward.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, P, ctypes.c_int, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ----------------------------------------------------------------- primitives

def philox(ctr, key):
    out = np.zeros(4, np.uint32)
    c, k = _c(ctr, np.uint32), _c(key, np.uint32)
    lib().orc_philox(_p(c), _p(k), _p(out))
    return out


def sample_indices(n, size, batch, seed, learner, rnd):
    """O2: uniform minibatch slot indices tau (absolute step numbers)."""
    tau = np.zeros(batch, np.int64)
    if lib().orc_sample_indices(n, size, batch, seed, learner, rnd, _p(tau)) != 0:
        raise ValueError("replay has no valid transition")
    return tau


def sample_indices_global(ns, capacity, batch, seed, learner, rnd):
    """f4 (R36): (shard, tau) per sample, uniform over the union of the shards' valid transitions.
    ns: n_j of every shard in ascending global learner id; shard = position in ns."""
    ns = np.ascontiguousarray(ns, dtype=np.int64)
    shard = np.zeros(batch, np.int32)
    tau = np.zeros(batch, np.int64)
    if lib().orc_sample_indices_global(len(ns), _p(ns), capacity, batch, seed, learner, rnd, _p(shard), _p(tau)) != 0:
        raise ValueError("global replay has no valid transition")
    return shard, tau


def gather_global(rings, shard, tau):
    """O3 per sample from the ring of its shard (f4): the same stacking as Ring.gather."""
    parts = [rings[int(q)].gather(np.array([t], np.int64)) for q, t in zip(shard, tau)]
    return tuple(np.concatenate([p[f] for p in parts]) for f in range(5))


def round_bf16(x):
    return lib().orc_round_bf16(float(x))


def param_count(n_actions):
    return int(lib().orc_param_count(n_actions))


def conv2d_fwd(x, w, b, stride):
    x, w = _c(x, np.float64), _c(w, np.float64)
    B, Cin, H, W = x.shape
    Cout, _, k, _ = w.shape
    OH, OW = (H - k) // stride + 1, (W - k) // stride + 1
    y = np.zeros((B, Cout, OH, OW))
    bb = None if b is None else _c(b, np.float64)
    lib().orc_conv2d_fwd(B, Cin, H, W, Cout, k, stride, _p(x), _p(w), _p(bb), _p(y))
    return y


def conv2d_bwd_data(dy, w, in_hw, stride):
    dy, w = _c(dy, np.float64), _c(w, np.float64)
    B, Cout = dy.shape[:2]
    _, Cin, k, _ = w.shape
    H, W = in_hw
    dx = np.zeros((B, Cin, H, W))
    lib().orc_conv2d_bwd_data(B, Cin, H, W, Cout, k, stride, _p(dy), _p(w), _p(dx))
    return dx


def conv2d_bwd_weight(dy, x, k, stride):
    dy, x = _c(dy, np.float64), _c(x, np.float64)
    B, Cin, H, W = x.shape
    Cout = dy.shape[1]
    dw = np.zeros((Cout, Cin, k, k))
    db = np.zeros(Cout)
    lib().orc_conv2d_bwd_weight(B, Cin, H, W, Cout, k, stride, _p(dy), _p(x), _p(dw), _p(db))
    return dw, db


def linear_fwd(x, w, b):
    x, w = _c(x, np.float64), _c(w, np.float64)
    B, K = x.shape
    N = w.shape[0]
    y = np.zeros((B, N))
    bb = None if b is None else _c(b, np.float64)
    lib().orc_linear_fwd(B, K, N, _p(x), _p(w), _p(bb), _p(y))
    return y


def linear_bwd_data(dy, w):
    dy, w = _c(dy, np.float64), _c(w, np.float64)
    B, N = dy.shape
    K = w.shape[1]
    dx = np.zeros((B, K))
    lib().orc_linear_bwd_data(B, K, N, _p(dy), _p(w), _p(dx))
    return dx


def linear_bwd_weight(dy, x):
    dy, x = _c(dy, np.float64), _c(x, np.float64)
    B, N = dy.shape
    K = x.shape[1]
    dw = np.zeros((N, K))
    db = np.zeros(N)
    lib().orc_linear_bwd_weight(B, K, N, _p(dy), _p(x), _p(dw), _p(db))
    return dw, db


# canonical parameter layout: (name, shape) in order
def param_shapes(n_actions):
    return [("W1", (32, 4, 8, 8)), ("b1", (32,)), ("W2", (64, 32, 4, 4)), ("b2", (64,)),
            ("W3", (64, 64, 3, 3)), ("b3", (64,)), ("W4", (512, 3136)), ("b4", (512,)),
            ("W5", (n_actions, 512)), ("b5", (n_actions,))]


def unflatten(theta, n_actions):
    out, off = {}, 0
    for name, shp in param_shapes(n_actions):
        n = int(np.prod(shp))
        out[name] = theta[off:off + n].reshape(shp)
        off += n
    return out


def acts_per_sample():
    return int(lib().orc_acts_per_sample())


def qnet_forward(theta, s, n_actions, mode="exact", want_z=False):
    """O4: Q(s,.;theta) for s u8 [B][4][84][84]. Returns (Q [B][nA], saved activations), plus the
    pre-activations z1..z4 (same layout, the values each ReLU decides on) if want_z."""
    theta = _c(theta, np.float64)
    s = _c(s, np.uint8)
    B = s.shape[0]
    Q = np.zeros((B, n_actions))
    acts = np.zeros((B, acts_per_sample()))
    zs = np.zeros((B, acts_per_sample())) if want_z else None
    lib().orc_qnet_forward(n_actions, B, _p(theta), _p(s), MODES[mode], _p(Q), _p(acts), _p(zs))
    return (Q, acts, zs) if want_z else (Q, acts)


def qnet_backward(theta, s, acts, dQ, n_actions, mode="exact"):
    """G = sum_b sum_a dQ[b,a] dQ(s_b,a)/dtheta (canonical layout)."""
    theta = _c(theta, np.float64)
    s = _c(s, np.uint8)
    dQ = _c(dQ, np.float64)
    G = np.zeros(theta.shape[0])
    lib().orc_qnet_backward(n_actions, s.shape[0], _p(theta), _p(s), _p(_c(acts, np.float64)), _p(dQ),
                            MODES[mode], _p(G))
    return G


def td_terms(Q, Qhat, a, r, d, gamma):
    """O5/O6 + Eq.2 with reading R3/R4.

    y_i = r_i if s_{i+1} terminal else r_i + gamma max_a' Qhat_i[a']   (Alg.1)
    delta_i = y_i - Q_i[a_i]; loss = mean delta^2 (Eq.1); l = mean |delta| (R7)
    dQ[i][a_i] = -clip(delta_i, -1, 1) / B  (dL/dQ of the Huber(1)-clipped per-sample loss)
    """
    Q = np.asarray(Q, np.float64)
    Qhat = np.asarray(Qhat, np.float64)
    B = Q.shape[0]
    y = np.zeros(B)
    delta = np.zeros(B)
    dQ = np.zeros_like(Q)
    for i in range(B):
        if d[i]:
            y[i] = float(r[i])
        else:
            y[i] = float(r[i]) + gamma * float(np.max(Qhat[i]))
        delta[i] = y[i] - Q[i, int(a[i])]
        dQ[i, int(a[i])] = -min(max(delta[i], -1.0), 1.0) / B
    loss = float(np.mean(delta ** 2))
    abs_loss = float(np.mean(np.abs(delta)))
    return y, delta, dQ, loss, abs_loss


@dataclasses.dataclass
class LossStats:
    """Running EMA mean / variance of the absolute DQN loss (reading R8)."""
    mu: float = 0.0
    var: float = 0.0
    count: int = 0

    def rejects(self, ell, k_sigma, warmup):
        return self.count >= warmup and ell > self.mu + k_sigma * np.sqrt(self.var)

    def update(self, ell, beta):
        if self.count == 0:
            self.mu, self.var = ell, 0.0
        else:
            e = ell - self.mu
            self.mu = self.mu + (1.0 - beta) * e
            self.var = beta * (self.var + (1.0 - beta) * e * e)
        self.count += 1


def is_stale(v0, base_version, max_delay):
    """discard gradients older than the threshold (reading R10)."""
    return max_delay >= 0 and (v0 - base_version) > max_delay


def rmsprop_apply(theta, m, v, g, lr, rho, eps):
    """Centered RMSProp (reading R2), elementwise, in place on fp64 arrays."""
    m *= rho
    m += (1.0 - rho) * g
    v *= rho
    v += (1.0 - rho) * g * g
    theta -= lr * g / np.sqrt(v - m * m + eps)


def adagrad_apply(theta, acc, g, lr, eps):
    """AdaGrad ("we used the AdaGrad update rule"; SPEC S:63 form)."""
    acc += g * g
    theta -= lr * g / (np.sqrt(acc) + eps)


def shard_bounds(P, n_shards, align=256):
    """Contiguous equal blocks of the padded vector ("split disjointly"; reading R26)."""
    unit = align * n_shards
    P_pad = (P + unit - 1) // unit * unit
    per = P_pad // n_shards
    return [(min(r * per, P), min((r + 1) * per, P)) for r in range(n_shards)]


def should_sync(version, last_sync, period):
    """R13: theta^- <- theta^+ iff V >= last + N (Alg.1)."""
    return version >= last_sync + period


# ----------------------------------------------------------------- replay ring

class Ring:
    """Frame ring of capacity C (R14): slot of step t is t mod C."""

    def __init__(self, capacity):
        self.C = int(capacity)
        self.frames = np.zeros((self.C, 84, 84), np.uint8)
        self.a = np.zeros(self.C, np.uint8)
        self.r = np.zeros(self.C, np.float32)
        self.d = np.zeros(self.C, np.uint8)
        self.n = 0

    @property
    def size(self):
        return min(self.n, self.C)

    def insert(self, frames, a, r, d):
        cnt = len(a)
        for i in range(cnt):
            slot = (self.n + i) % self.C
            self.frames[slot] = frames[i]
            self.a[slot] = a[i]
            self.r[slot] = r[i]
            self.d[slot] = d[i]
        self.n += cnt

    def stack(self, t):
        out = np.zeros((4, 84, 84), np.uint8)
        lib().orc_stack(self.C, self.n, _p(self.frames), _p(self.d), t, _p(out))
        return out

    def gather(self, tau):
        B = len(tau)
        tau = _c(tau, np.int64)
        s = np.zeros((B, 4, 84, 84), np.uint8)
        s2 = np.zeros_like(s)
        a = np.zeros(B, np.uint8)
        r = np.zeros(B, np.float32)
        d = np.zeros(B, np.uint8)
        lib().orc_gather(self.C, self.n, _p(self.frames), _p(self.a), _p(self.r), _p(self.d), B, _p(tau),
                         _p(s), _p(s2), _p(a), _p(r), _p(d))
        return s, s2, a, r, d


# ----------------------------------------------------------------- the round

@dataclasses.dataclass
class Config:
    n_actions: int = 4
    batch: int = 32
    gamma: float = 0.99
    capacity: int = 10_000
    learners: tuple = (0,)          # global learner ids, ascending
    lr: float = 2.5e-4
    rms_rho: float = 0.95
    rms_eps: float = 0.01
    optimizer: str = "rmsprop"      # "rmsprop" (graded, R1) or "adagrad"
    ada_eps: float = 1e-8
    target_period: int = 100        # N (Alg.1; P:188 uses 60K)
    max_staleness: int = -1         # <0 disables
    outlier_enabled: bool = True
    outlier_warmup: int = 100
    outlier_k: float = 3.0
    outlier_beta: float = 0.999
    min_replay: int = 1
    seed_sample: int = 1507
    mode: str = "exact"             # "exact" (fp64) or "bf16" (emulates the GPU rounding points)
    n_shards: int = 1
    ps_mode: str = "aggregate"      # "aggregate": one step on the mean of the accepted gradients (R12);
                                    # "per_message": NEXT row f1, one optimizer step per accepted
                                    # message in ascending learner id, V += 1 each (R32)
    replay_mode: str = "local"      # "local": each learner samples its own ring (P:140 first form);
                                    # "global": NEXT row f4, uniform over the union of all learners'
                                    # rings as of the round's start (P:140 second form; R36)


@dataclasses.dataclass
class LearnerState:
    ring: Ring
    theta_minus: np.ndarray
    last_sync: int = 0
    stats: LossStats = dataclasses.field(default_factory=LossStats)


class GorilaOracle:
    """Deterministic fixed-order, fixed-staleness rounds."""

    def __init__(self, cfg: Config, theta0):
        self.cfg = cfg
        theta0 = np.asarray(theta0, np.float64)
        assert theta0.shape[0] == param_count(cfg.n_actions)
        self.theta = theta0.copy()
        self.m = np.zeros_like(self.theta)
        self.v = np.zeros_like(self.theta)
        self.V = 0
        # theta^- = theta at init (Alg.1)
        self.learners = {j: LearnerState(Ring(cfg.capacity), theta0.copy()) for j in cfg.learners}
        self.history = {}  # round -> (theta, V) at the start of that round

    def insert(self, j, frames, a, r, d):
        self.learners[j].ring.insert(frames, a, r, d)

    def round(self, k, staleness=None, acts_hook=None):
        """One round O1-O12. acts_hook (test teacher forcing, SURVEY §8(c) parity protocol):
        acts_hook(j, acts, zs) -> the activations learner j's backward (O8) takes instead of its own
        O4 activations; None = the oracle's own."""
        cfg = self.cfg
        staleness = staleness or {}
        self.history[k] = (self.theta.copy(), self.V)
        V0 = self.V
        per = {}
        G_sum = np.zeros_like(self.theta)
        n_acc = 0
        messages = []  # learners with a message (not rejected), ascending id (f1)
        for j in sorted(self.learners):
            L = self.learners[j]
            # O1
            k_src = max(k - int(staleness.get(j, 0)), 0)
            theta_j, b_j = self.history[k_src]
            info = {"base_version": b_j, "not_ready": False, "rejected_outlier": False,
                    "stale": False, "accepted": False}
            # O2
            if L.ring.size - 1 < max(1, cfg.min_replay):
                info["not_ready"] = True
                per[j] = info
                continue
            if cfg.replay_mode == "global":  # f4: draw (shard, tau) from the union, gather from that ring
                ids = sorted(self.learners)
                shard, tau = sample_indices_global([self.learners[q].ring.n for q in ids], cfg.capacity,
                                                   cfg.batch, cfg.seed_sample, j, k)
                s, s2, a, r, d = gather_global([self.learners[q].ring for q in ids], shard, tau)
            else:
                shard = None
                tau = sample_indices(L.ring.n, L.ring.size, cfg.batch, cfg.seed_sample, j, k)
                # O3
                s, s2, a, r, d = L.ring.gather(tau)
            # O4
            Q, acts, zs = qnet_forward(theta_j, s, cfg.n_actions, cfg.mode, want_z=True)
            if acts_hook is not None:
                acts = acts_hook(j, acts, zs)
            Qhat, _ = qnet_forward(L.theta_minus, s2, cfg.n_actions, cfg.mode)
            # O5, O6
            y, delta, dQ, loss, ell = td_terms(Q, Qhat, a, r, d, cfg.gamma)
            # O7: decide on pre-update stats, then update with every batch
            rejected = bool(cfg.outlier_enabled and L.stats.rejects(ell, cfg.outlier_k, cfg.outlier_warmup))
            thr = L.stats.mu + cfg.outlier_k * np.sqrt(L.stats.var)
            stats_count_before = L.stats.count
            L.stats.update(ell, cfg.outlier_beta)
            # O9 (per-message mode: judged at the PS, message by message, below)
            stale = is_stale(V0, b_j, cfg.max_staleness) if cfg.ps_mode != "per_message" else False
            info.update(tau=tau, shard=shard, Q=Q, Qhat=Qhat, y=y, delta=delta, loss=loss, abs_loss=ell,
                        threshold=thr, stats_count_before=stats_count_before,
                        rejected_outlier=rejected, stale=stale, mu=L.stats.mu, var=L.stats.var,
                        a=a, r=r, d=d)
            # O8
            if not rejected:
                G = qnet_backward(theta_j, s, acts, dQ, cfg.n_actions, cfg.mode)
                info["G"] = G
                if cfg.ps_mode == "per_message":
                    messages.append(j)
                elif not stale:
                    info["accepted"] = True
                    G_sum += G
                    n_acc += 1
            per[j] = info
        synced = {j: False for j in self.learners}
        # f1 (R32, R37): the messages arrive at the PS one by one in ascending learner id. Each is judged
        # against the PS version when it arrives ("older than a threshold"; V counts the
        # updates applied so far), applied as its own optimizer step if fresh (V += 1), and
        # after every step each learner's target net syncs if V >= last + N ("after every N
        # gradient updates in the central parameter server") -- possibly inside the round.
        if cfg.ps_mode == "per_message":
            V = V0
            for j in messages:
                info = per[j]
                info["stale"] = is_stale(V, info["base_version"], cfg.max_staleness)
                info["version_at_arrival"] = V
                if info["stale"]:
                    continue
                info["accepted"] = True
                G = info["G"]
                for lo, hi in shard_bounds(len(self.theta), cfg.n_shards):
                    if cfg.optimizer == "rmsprop":
                        rmsprop_apply(self.theta[lo:hi], self.m[lo:hi], self.v[lo:hi], G[lo:hi],
                                      cfg.lr, cfg.rms_rho, cfg.rms_eps)
                    else:
                        adagrad_apply(self.theta[lo:hi], self.v[lo:hi], G[lo:hi], cfg.lr, cfg.ada_eps)
                V += 1
                n_acc += 1
                for i in sorted(self.learners):
                    Li = self.learners[i]
                    if should_sync(V, Li.last_sync, cfg.target_period):
                        Li.theta_minus = self.theta.copy()
                        Li.last_sync = V
                        synced[i] = True
            self.V = V
        # O10 (one PS step per round on the mean of accepted gradients; R12, R25)
        elif n_acc > 0:
            g = G_sum / n_acc
            for lo, hi in shard_bounds(len(self.theta), cfg.n_shards):
                if cfg.optimizer == "rmsprop":
                    rmsprop_apply(self.theta[lo:hi], self.m[lo:hi], self.v[lo:hi], g[lo:hi],
                                  cfg.lr, cfg.rms_rho, cfg.rms_eps)
                else:
                    adagrad_apply(self.theta[lo:hi], self.v[lo:hi], g[lo:hi], cfg.lr, cfg.ada_eps)
            self.V = V0 + n_acc
        # O11 is implicit: the next round reads self.theta / self.V (history)
        # O12 (per-message mode: taken after every step above)
        for j in sorted(self.learners):
            L = self.learners[j]
            if cfg.ps_mode == "per_message":
                continue
            synced[j] = should_sync(self.V, L.last_sync, cfg.target_period)
            if synced[j]:
                L.theta_minus = self.theta.copy()
                L.last_sync = self.V
        return {"learners": per, "n_accepted": n_acc, "version_before": V0, "version_after": self.V,
                "synced": synced}


# ----------------------------------------------------------------- NEXT row f3: acting
# Alg.1 P:118 "select an action a_t with the epsilon-greedy policy on Q(s; theta)"; epsilon
# annealed linearly from 1 to its final value over the first million updates.
TAG_ACT = 5


def epsilon(global_step, eps_final, anneal_steps):
    """Linear anneal from 1 to eps_final over anneal_steps global steps, then constant."""
    if anneal_steps <= 0 or global_step >= anneal_steps:
        return float(eps_final)
    return 1.0 - (1.0 - float(eps_final)) * (float(global_step) / float(anneal_steps))


def act_draws(n, actor_id, global_step, seed):
    """Per state i: Philox4x32-10(ctr = {i, actor, step lo, (step hi & 0xffffff) | TAG_ACT << 24},
    key = {seed lo, seed hi}) -> (u = x0 * 2^-32 for the explore test, x1 for the random action)."""
    key = np.array([seed & 0xffffffff, (seed >> 32) & 0xffffffff], np.uint32)
    out = []
    for i in range(n):
        ctr = np.array([i, actor_id & 0xffffffff, global_step & 0xffffffff,
                        ((global_step >> 32) & 0xffffff) | (TAG_ACT << 24)], np.uint32)
        x = philox(ctr, key)
        out.append((int(x[0]), int(x[1])))
    return out


def act(theta, s, n_actions, mode, global_step, actor_id, eps_final, anneal_steps, seed):
    """epsilon-greedy actions on Q(s; theta): explore iff x0 < eps * 2^32 (compared in fp64 on the
    integer x0), then a = floor(x1 * nA / 2^32); else the argmax with the lowest index on ties.
    Returns (actions, Q)."""
    Q, _ = qnet_forward(theta, s, n_actions, mode)
    eps = epsilon(global_step, eps_final, anneal_steps)
    acts = np.zeros(len(s), np.int32)
    for i, (x0, x1) in enumerate(act_draws(len(s), actor_id, global_step, seed)):
        if float(x0) < eps * 4294967296.0:
            acts[i] = (x1 * n_actions) >> 32
        else:
            acts[i] = int(np.argmax(Q[i]))  # numpy argmax: first maximal index
    return acts, Q
