"""Thin ctypes binding of the C-ABI in include/gorila.h (argument marshalling only).

Every step of the learner update runs in libgorila.so's sm_100a kernels; this
module only converts Python / numpy / torch arguments to pointers. There is no
CPU fallback: if the library is missing or fails to load, ``load()`` raises.
PyTorch provides the device workspace and the stream (plumbing only).
"""
import ctypes
import os

import numpy as np

from . import _build

_lib = None

GORILA_MATH_FP32 = 0
GORILA_MATH_BF16 = 2
GORILA_OPT_RMSPROP = 0
GORILA_OPT_ADAGRAD = 1
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_SHAPE", 3: "E_RANGE", 4: "E_NOT_READY", 5: "E_CUDA", 6: "E_NCCL",
          7: "E_OOM"}


class GorilaError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("n_actions", ctypes.c_int32), ("batch", ctypes.c_int32), ("gamma", ctypes.c_float),
                ("replay_capacity", ctypes.c_int64), ("n_learners_local", ctypes.c_int32),
                ("learner_id_base", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("stream", ctypes.c_void_p), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_uint64), ("optimizer", ctypes.c_int32), ("lr", ctypes.c_float),
                ("rms_rho", ctypes.c_float), ("rms_eps", ctypes.c_float), ("ada_eps", ctypes.c_float),
                ("target_period", ctypes.c_int64), ("max_staleness", ctypes.c_int64),
                ("outlier_enabled", ctypes.c_int32), ("outlier_warmup", ctypes.c_int32),
                ("outlier_k", ctypes.c_float), ("outlier_beta", ctypes.c_double), ("min_replay", ctypes.c_int64),
                ("seed", ctypes.c_uint64), ("math", ctypes.c_int32), ("history", ctypes.c_int32),
                ("theta0", ctypes.c_void_p), ("ps_mode", ctypes.c_int32),
                ("replay_mode", ctypes.c_int32)]


class LearnerInfo(ctypes.Structure):
    _fields_ = [("loss", ctypes.c_float), ("abs_loss", ctypes.c_float), ("mu", ctypes.c_double),
                ("var", ctypes.c_double), ("threshold", ctypes.c_double), ("base_version", ctypes.c_uint64),
                ("stats_count", ctypes.c_uint32), ("not_ready", ctypes.c_uint8), ("rejected_outlier", ctypes.c_uint8),
                ("stale", ctypes.c_uint8), ("accepted", ctypes.c_uint8)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class RoundInfo(ctypes.Structure):
    _fields_ = [("n_accepted", ctypes.c_uint32), ("pad_", ctypes.c_uint32), ("version_before", ctypes.c_uint64),
                ("version_after", ctypes.c_uint64)]


class AsyncStats(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_uint64), ("sent", ctypes.c_uint64), ("fresh", ctypes.c_uint64),
                ("stale", ctypes.c_uint64), ("rejected", ctypes.c_uint64), ("version_after", ctypes.c_uint64),
                ("max_delay", ctypes.c_uint64), ("mean_delay", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ["gorila_param_count", "gorila_workspace_bytes", "gorila_init", "gorila_destroy", "gorila_last_error",
           "replay_insert", "replay_sample", "replay_sample_shards", "learner_step", "ps_apply_shard", "sync_target", "gorila_get_state",
           "gorila_set_state", "gorila_get_learner_state", "gorila_set_learner_state", "gorila_get_grad",
           "gorila_get_q", "gorila_get_activation", "gorila_act", "gorila_kernel_launches", "gorila_profile_enable", "gorila_profile_read",
           "gorila_profile_phase_count", "gorila_profile_phase_name", "gorila_nccl_unique_id", "gorila_round",
           "gorila_round_async", "gorila_round_post", "gorila_round_fetch",
           "gorila_bench_phase", "gorila_debug_trace", "gorila_debug_trace_tiles", "gorila_capture_activations",
           "gorila_get_learner_activation", "gorila_peer_record", "gorila_peer_connect", "gorila_async_run"]


def load(build_if_missing=True):
    """Load libgorila.so (building it in-tree if absent). Raises if it cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and _build.stale():
        _build.build()
    so = os.environ.get("GORILA_LIB", _build.SO)  # diagnostics builds (e.g. libgorila_trace.so)
    if not os.path.exists(so):
        raise RuntimeError(f"libgorila.so missing at {so}: run __graft_entry__.build()")
    L = ctypes.CDLL(so)
    P, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    L.gorila_param_count.argtypes = [i32]
    L.gorila_param_count.restype = i64
    L.gorila_workspace_bytes.argtypes = [ctypes.POINTER(Config)]
    L.gorila_workspace_bytes.restype = u64
    L.gorila_init.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(P)]
    L.gorila_destroy.argtypes = [P]
    L.gorila_last_error.restype = ctypes.c_char_p
    L.replay_insert.argtypes = [P, i32, i64, P, P, P, P, i32]
    L.replay_sample.argtypes = [P, i32, u64, P, P, P, P, P, P]
    L.replay_sample_shards.argtypes = [P, P]
    L.learner_step.argtypes = [P, P, i32, u64, P, P]
    L.ps_apply_shard.argtypes = [P, u64, P]
    L.sync_target.argtypes = [P, P, i32, i32, P]
    L.gorila_get_state.argtypes = [P, P, P, P, P]
    L.gorila_set_state.argtypes = [P, P, P, P, u64]
    L.gorila_get_learner_state.argtypes = [P, i32, P, P]
    L.gorila_set_learner_state.argtypes = [P, i32, P, P]
    L.gorila_get_grad.argtypes = [P, P]
    L.gorila_get_q.argtypes = [P, i32, P, P]
    L.gorila_get_activation.argtypes = [P, i32, P, u64]
    L.gorila_capture_activations.argtypes = [P, i32]
    L.gorila_peer_record.argtypes = [P, P]
    L.gorila_peer_connect.argtypes = [P, P, i32]
    L.gorila_async_run.argtypes = [P, P, i32, i64, u64, i32, ctypes.POINTER(AsyncStats)]
    L.gorila_get_learner_activation.argtypes = [P, i32, i32, P, u64]
    L.gorila_round_post.argtypes = [P, P, i32, u64, P]
    L.gorila_round_fetch.argtypes = [P, u64, P, P, P]
    L.gorila_act.argtypes = [P, P, i32, u64, u64, ctypes.c_double, i64, i32, P, P]
    L.gorila_kernel_launches.argtypes = [P]
    L.gorila_kernel_launches.restype = u64
    L.gorila_profile_enable.argtypes = [P, i32]
    L.gorila_profile_read.argtypes = [P, P, i32, P]
    L.gorila_profile_phase_count.restype = i32
    L.gorila_profile_phase_name.argtypes = [i32]
    L.gorila_profile_phase_name.restype = ctypes.c_char_p
    L.gorila_nccl_unique_id.argtypes = [P]
    L.gorila_round.argtypes = [P, P, i32, u64, P, P, P, P]
    L.gorila_round_async.argtypes = [P, P, i32, u64, P, P, P, P]
    L.gorila_bench_phase.argtypes = [P, i32, i32, i32, P]
    L.gorila_debug_trace.argtypes = [P]
    L.gorila_debug_trace_tiles.argtypes = [P]
    _lib = L
    return L


def _check(st):
    if st != 0:
        raise GorilaError(st, _lib.gorila_last_error().decode())


def nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (rank 0; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().gorila_nccl_unique_id(buf))
    return buf.raw


def phase_names():
    L = load()
    return [L.gorila_profile_phase_name(i).decode() for i in range(L.gorila_profile_phase_count())]


def param_count(n_actions):
    return int(load().gorila_param_count(n_actions))


def _ptr(x):
    """host numpy array or torch tensor -> (pointer, is_device)."""
    if x is None:
        return None, False
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data, False
    # torch tensor
    assert x.is_contiguous()
    return x.data_ptr(), bool(x.is_cuda)


class Gorila:
    """One rank's learner / parameter-server context (see include/gorila.h)."""

    def __init__(self, n_actions=18, batch=32, gamma=0.99, replay_capacity=1_000_000, n_learners_local=1,
                 learner_id_base=0, rank=0, world=1, nccl_unique_id=None, stream=None, theta0=None,
                 optimizer="rmsprop", lr=2.5e-4, rms_rho=0.95, rms_eps=0.01, ada_eps=1e-8, target_period=100,
                 max_staleness=-1, outlier_enabled=True, outlier_warmup=100, outlier_k=3.0, outlier_beta=0.999,
                 min_replay=1, seed=1507, math="bf16", history=2, device=None, ps_mode="aggregate",
                 replay_mode="local"):
        import torch
        L = load()
        self.torch = torch
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        # a dedicated stream by default (the legacy default stream cannot be graph-captured)
        self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        self.n_actions, self.batch, self.L = n_actions, batch, n_learners_local
        self.math = math
        self.P = param_count(n_actions)
        theta0 = np.ascontiguousarray(theta0, dtype=np.float32)
        assert theta0.shape == (self.P,)
        self._id = None
        if nccl_unique_id is not None:
            self._id = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
        cfg = Config(n_actions=n_actions, batch=batch, gamma=gamma, replay_capacity=replay_capacity,
                     n_learners_local=n_learners_local, learner_id_base=learner_id_base, rank=rank, world=world,
                     nccl_unique_id=ctypes.cast(self._id, ctypes.c_void_p) if self._id is not None else None,
                     stream=self.stream.cuda_stream, workspace=None, workspace_bytes=0,
                     optimizer={"rmsprop": 0, "adagrad": 1}[optimizer], lr=lr, rms_rho=rms_rho, rms_eps=rms_eps,
                     ada_eps=ada_eps, target_period=target_period, max_staleness=max_staleness,
                     outlier_enabled=int(outlier_enabled), outlier_warmup=outlier_warmup, outlier_k=outlier_k,
                     outlier_beta=outlier_beta, min_replay=min_replay, seed=seed,
                     ps_mode={"aggregate": 0, "per_message": 1, "async": 2}[ps_mode],
                     replay_mode={"local": 0, "global": 1}[replay_mode],
                     math={"fp32": 0, "bf16": 2}[math], history=history, theta0=theta0.ctypes.data)
        nbytes = int(L.gorila_workspace_bytes(ctypes.byref(cfg)))
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        cfg.workspace = self.workspace.data_ptr()
        cfg.workspace_bytes = nbytes
        self.cfg = cfg
        h = ctypes.c_void_p()
        _check(L.gorila_init(ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h
        if world > 1 and nccl_unique_id is None:
            self._connect_peers()
        self._info = (LearnerInfo * max(1, n_learners_local))()

    def _connect_peers(self):
        """Caller-bootstrapped peer mappings (include/gorila.h gorila_peer_connect): the 128-byte
        records all-gathered over torch.distributed's default process group (any backend: gloo works
        for several ranks sharing one GPU); every rank raises if any rank failed."""
        import torch.distributed as dist
        L = load()
        rec = ctypes.create_string_buffer(128)
        st = L.gorila_peer_record(self.h, rec)
        recs = [None] * dist.get_world_size()
        dist.all_gather_object(recs, rec.raw if st == 0 else None)
        ok = all(r is not None for r in recs)
        st2 = L.gorila_peer_connect(self.h, ctypes.create_string_buffer(b"".join(recs), 128 * len(recs)),
                                    len(recs)) if ok else 1
        verdict = [None] * dist.get_world_size()
        dist.all_gather_object(verdict, st2 == 0)
        if not all(verdict):
            msg = L.gorila_last_error().decode() if st2 != 0 else "a peer failed to connect"
            raise GorilaError(st2 if st2 != 0 else 5, "peer mapping failed: " + msg)

    def close(self):
        if self.h:
            load().gorila_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- replay
    def replay_insert(self, learner, frames, actions, rewards, terminals):
        count = int(frames.shape[0])
        fp, dev = _ptr(frames)
        if dev:  # device inputs produced on torch's current stream: order our stream after it
            self.stream.wait_stream(self.torch.cuda.current_stream(self.device))
        ap, _ = _ptr(actions)
        rp, _ = _ptr(rewards)
        dp, _ = _ptr(terminals)
        _check(load().replay_insert(self.h, learner, count, fp, ap, rp, dp, int(dev)))
        if dev:  # the copies read the sources on our stream: the caller's stream may reuse them after
            self.torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def replay_sample_shards(self):
        """Shard (global learner id) of each sample of the most recent draw (f4)."""
        out = np.zeros(self.batch, np.int32)
        _check(load().replay_sample_shards(self.h, out.ctypes.data))
        return out

    def replay_sample(self, learner, rnd):
        B = self.batch
        idx = np.zeros(B, np.int64)
        s = np.zeros((B, 4, 84, 84), np.uint8)
        s2 = np.zeros_like(s)
        a = np.zeros(B, np.uint8)
        r = np.zeros(B, np.float32)
        d = np.zeros(B, np.uint8)
        _check(load().replay_sample(self.h, learner, rnd, idx.ctypes.data, s.ctypes.data, s2.ctypes.data,
                                    a.ctypes.data, r.ctypes.data, d.ctypes.data))
        return {"tau": idx, "s": s, "s2": s2, "a": a, "r": r, "d": d}

    # ---------------------------------------------------------------- the round
    def learner_step(self, learners, rnd, staleness=None, want_info=True):
        ids = np.ascontiguousarray(learners, dtype=np.int32)
        st = None if staleness is None else np.ascontiguousarray(staleness, dtype=np.int32)
        info = self._info if want_info else None
        _check(load().learner_step(self.h, ids.ctypes.data, len(ids), rnd, None if st is None else st.ctypes.data,
                                   ctypes.cast(info, ctypes.c_void_p) if info is not None else None))
        if not want_info:
            return None
        self.stream.synchronize()
        return [self._info[i].as_dict() for i in range(len(ids))]

    def learner_step_async(self, learners_arr, rnd, staleness_arr=None):
        """No host sync, no info copy (throughput path). learners_arr: int32 numpy array."""
        _check(load().learner_step(self.h, learners_arr.ctypes.data, len(learners_arr), rnd,
                                   None if staleness_arr is None else staleness_arr.ctypes.data, None))

    def round(self, learners_arr, rnd, staleness_arr=None, want_info=False):
        """learner_step + ps_apply_shard + sync_target as one (graph-replayed) round."""
        if not want_info:
            _check(load().gorila_round(self.h, learners_arr.ctypes.data, len(learners_arr), rnd,
                                       None if staleness_arr is None else staleness_arr.ctypes.data,
                                       None, None, None))
            return None
        ri = RoundInfo()
        synced = np.zeros(len(learners_arr), np.uint8)
        _check(load().gorila_round(self.h, learners_arr.ctypes.data, len(learners_arr), rnd,
                                   None if staleness_arr is None else staleness_arr.ctypes.data,
                                   ctypes.cast(self._info, ctypes.c_void_p), ctypes.byref(ri), synced.ctypes.data))
        return ([self._info[i].as_dict() for i in range(len(learners_arr))],
                {"n_accepted": ri.n_accepted, "version_before": ri.version_before,
                 "version_after": ri.version_after}, synced.astype(bool))

    def round_async(self, learners_arr, rnd, staleness_arr=None):
        """gorila_round_post: the round's result is stored by its own last kernel into the library's
        pinned result ring; returns a handle for round_result (read it while later rounds run)."""
        _check(load().gorila_round_post(self.h, learners_arr.ctypes.data, len(learners_arr), rnd,
                                        None if staleness_arr is None else staleness_arr.ctypes.data))
        return (rnd, len(learners_arr))

    def round_result(self, handle):
        """gorila_round_fetch for a round_async handle (polls host memory, no CUDA call); returns
        (learner infos, round info, synced) like round()."""
        rnd, n = handle
        infos = (LearnerInfo * n)()
        ri = RoundInfo()
        synced = np.zeros(n, np.uint8)
        _check(load().gorila_round_fetch(self.h, rnd, ctypes.cast(infos, ctypes.c_void_p), ctypes.byref(ri),
                                         synced.ctypes.data))
        return ([infos[i].as_dict() for i in range(n)],
                {"n_accepted": ri.n_accepted, "version_before": ri.version_before, "version_after": ri.version_after},
                synced.astype(bool))

    def ps_apply_shard(self, rnd, want_info=True):
        ri = RoundInfo() if want_info else None
        _check(load().ps_apply_shard(self.h, rnd, ctypes.byref(ri) if ri is not None else None))
        if ri is None:
            return None
        return {"n_accepted": ri.n_accepted, "version_before": ri.version_before, "version_after": ri.version_after}

    def sync_target(self, learners, force=False, want_info=True):
        ids = np.ascontiguousarray(learners, dtype=np.int32)
        out = np.zeros(len(ids), np.uint8)
        _check(load().sync_target(self.h, ids.ctypes.data, len(ids), int(force),
                                  out.ctypes.data if want_info else None))
        if not want_info:
            return None
        self.stream.synchronize()
        return out.astype(bool)

    # ---------------------------------------------------------------- state
    def get_state(self):
        th = np.zeros(self.P, np.float32)
        m = np.zeros(self.P, np.float32)
        v = np.zeros(self.P, np.float32)
        ver = ctypes.c_uint64()
        _check(load().gorila_get_state(self.h, th.ctypes.data, m.ctypes.data, v.ctypes.data, ctypes.byref(ver)))
        return th, m, v, ver.value

    def set_state(self, theta, m=None, v=None, version=0):
        th = np.ascontiguousarray(theta, np.float32)
        mm = None if m is None else np.ascontiguousarray(m, np.float32)
        vv = None if v is None else np.ascontiguousarray(v, np.float32)
        _check(load().gorila_set_state(self.h, th.ctypes.data, None if mm is None else mm.ctypes.data,
                                       None if vv is None else vv.ctypes.data, version))

    def get_learner_state(self, learner):
        tm = np.zeros(self.P, np.float32)
        st = np.zeros(4, np.float64)
        _check(load().gorila_get_learner_state(self.h, learner, tm.ctypes.data, st.ctypes.data))
        return tm, {"mu": st[0], "var": st[1], "count": int(st[2]), "last_sync": int(st[3])}

    def set_learner_state(self, learner, theta_minus=None, mu=0.0, var=0.0, count=0, last_sync=0):
        tm = None if theta_minus is None else np.ascontiguousarray(theta_minus, np.float32)
        st = np.array([mu, var, count, last_sync], np.float64)
        _check(load().gorila_set_learner_state(self.h, learner, None if tm is None else tm.ctypes.data,
                                               st.ctypes.data))

    def get_grad(self):
        g = np.zeros(self.P, np.float32)
        _check(load().gorila_get_grad(self.h, g.ctypes.data))
        return g

    def get_q(self, learner):
        q = np.zeros((self.batch, self.n_actions), np.float32)
        qh = np.zeros_like(q)
        _check(load().gorila_get_q(self.h, learner, q.ctypes.data, qh.ctypes.data))
        return q, qh

    _ACT = {"s": (0, (84, 84, 4)), "a1": (1, (20, 20, 32)), "a2": (2, (9, 9, 64)), "a3": (3, (7, 7, 64)),
            "a4": (4, (512,)), "g1": (5, (20, 20, 32)), "g2": (6, (9, 9, 64)), "g3": (7, (7, 7, 64)),
            "g4": (8, (512,))}

    def get_activation(self, name):
        """Intermediate tensor of the last learner step as float32 (bf16 mode values widened)."""
        which, shp = self._ACT[name]
        bf = self.math == "bf16" and name != "a4"
        out = np.zeros((self.batch,) + shp, np.uint16 if bf else np.float32)
        _check(load().gorila_get_activation(self.h, which, out.ctypes.data, out.nbytes))
        return (out.astype(np.uint32) << 16).view(np.float32) if bf else out

    def async_run(self, learners, steps, round0=0, server_blocks=0):
        """NEXT row f2 (ps_mode="async"): `steps` asynchronous learner steps per listed learner while the
        persistent shard server applies their messages; returns the counts (include/gorila.h)."""
        arr = np.ascontiguousarray(learners, np.int32)
        st = AsyncStats()
        _check(load().gorila_async_run(self.h, arr.ctypes.data, len(arr), int(steps), int(round0), int(server_blocks),
                                       ctypes.byref(st)))
        return st.as_dict()

    def capture_activations(self, on=True):
        """Parity diagnostics: keep every learner's a1..a4 of each later learner step."""
        _check(load().gorila_capture_activations(self.h, int(bool(on))))

    def get_learner_activation(self, learner, name):
        """Learner `learner`'s a1..a4 of its last step (capture_activations must be on), as float32."""
        which, shp = self._ACT[name]
        bf = self.math == "bf16" and name != "a4"
        out = np.zeros((self.batch,) + shp, np.uint16 if bf else np.float32)
        _check(load().gorila_get_learner_activation(self.h, learner, which, out.ctypes.data, out.nbytes))
        return (out.astype(np.uint32) << 16).view(np.float32) if bf else out

    def act(self, states, global_step, actor_id=0, eps_final=0.1, anneal_steps=1_000_000):
        """NEXT row f3: epsilon-greedy actions (and Q) for stacked u8 states [n][4][84][84] (host
        numpy or device tensor) on the latest theta^+ replica."""
        n = int(states.shape[0])
        sp, dev = _ptr(states)
        if dev:
            self.stream.wait_stream(self.torch.cuda.current_stream(self.device))
        acts = np.zeros(n, np.int32)
        q = np.zeros((n, self.n_actions), np.float32)
        _check(load().gorila_act(self.h, sp, n, int(global_step), int(actor_id), float(eps_final), int(anneal_steps),
                                 int(dev), acts.ctypes.data, q.ctypes.data))
        return acts, q

    def kernel_launches(self):
        return int(load().gorila_kernel_launches(self.h))

    # ---------------------------------------------------------------- diagnostics
    def profile_enable(self, on=True):
        _check(load().gorila_profile_enable(self.h, int(on)))

    def profile_read(self):
        """{phase: summed ms} since the last read, and the number of learner steps covered."""
        names = phase_names()
        ms = np.zeros(len(names), np.float64)
        n = ctypes.c_uint64()
        _check(load().gorila_profile_read(self.h, ms.ctypes.data, len(names), ctypes.byref(n)))
        return dict(zip(names, ms.tolist())), int(n.value)

    def bench_phase(self, phase_name, learner=0, iters=200):
        """Mean device microseconds of one phase's kernels, re-launched back to back (diagnostics)."""
        idx = phase_names().index(phase_name)
        us = ctypes.c_double()
        _check(load().gorila_bench_phase(self.h, learner, idx, iters, ctypes.byref(us)))
        return us.value
