"""world_size-2 gloo test (CPU) of the sharded parameter-server protocol.

Each process is one rank with one learner (bundled mode). Per round, exactly as the
C-ABI library does it over NCCL: the rank's gradient sum G (internal flat vector padded to
W*q, q = ceil(P/W) rounded to 64) and its accepted count (one slot per destination shard)
are reduce-scattered onto the owning shard; the owner applies the optimizer to its slice
with the mean of the accepted gradients (R12, R25); the slices are all-gathered; V
advances by the global accepted count. The result must equal the single-process oracle
with both learners (ascending ids) on one parameter server.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth

NA, B, C, ROUNDS, W = 4, 8, 400, 3, 2


def _cfg(learners, n_shards=1):
    return O.Config(n_actions=NA, batch=B, capacity=C, learners=learners, outlier_warmup=1, n_shards=n_shards)


def _fill(orc, j):
    f = synth.frames(synth.SEED_DATA, j, 0, C)
    a, r, d = synth.meta(synth.SEED_DATA, j, 0, C, NA)
    orc.insert(j, f, a, r, d)


def _rank_main(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    theta0 = synth.theta0(NA)
    P = theta0.shape[0]
    q = ((P + W - 1) // W + 63) // 64 * 64
    # this rank's learner: per-learner parts of the round come from the oracle's own round
    local = O.GorilaOracle(_cfg((rank,)), theta0)
    _fill(local, rank)
    theta = torch.zeros(W * q, dtype=torch.float64)
    theta[:P] = torch.from_numpy(theta0.astype(np.float64))
    m = torch.zeros(q, dtype=torch.float64)
    v = torch.zeros(q, dtype=torch.float64)
    V = 0
    lo = rank * q
    for k in range(ROUNDS):
        # learner side: the oracle's learner computations on the current replica
        local.theta = theta[:P].numpy().copy()
        local.V = V
        info = local.round(k)["learners"][rank]
        g = torch.zeros(W * q, dtype=torch.float64)
        if info["accepted"]:
            g[:P] = torch.from_numpy(info["G"])
        counts = torch.full((W,), float(info["accepted"]), dtype=torch.float64)
        # grouped reduce-scatter: gradient slices + count slots onto the owners
        g_slice = torch.zeros(q, dtype=torch.float64)
        dist.reduce_scatter(g_slice, list(g.split(q)))
        n_acc = torch.zeros(1, dtype=torch.float64)
        dist.reduce_scatter(n_acc, list(counts.split(1)))
        # owner applies the optimizer to its slice with the mean of the accepted gradients
        th_slice = theta[lo:lo + q].clone()
        if n_acc.item() > 0:
            n_real = max(0, min(q, P - lo))
            ts, ms, vs = th_slice[:n_real].numpy(), m[:n_real].numpy(), v[:n_real].numpy()
            O.rmsprop_apply(ts, ms, vs, (g_slice[:n_real] / n_acc.item()).numpy(), 2.5e-4, 0.95, 0.01)
        gathered = [torch.zeros(q, dtype=torch.float64) for _ in range(W)]
        dist.all_gather(gathered, th_slice)
        theta = torch.cat(gathered)
        V += int(n_acc.item())
        # target sync is local: every rank holds the full theta+ (R13)
        L = local.learners[rank]
        L.theta_minus = theta[:P].numpy().copy() if O.should_sync(V, L.last_sync, 100) else L.theta_minus
    if rank == 0:
        out.put((theta[:P].numpy(), V))
    dist.destroy_process_group()


def test_sharded_ps_equals_single_server():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_rank_main, args=(r, port, out)) for r in range(W)]
    for p in procs:
        p.start()
    theta_w, V_w = out.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = O.GorilaOracle(_cfg((0, 1)), synth.theta0(NA))
    _fill(ref, 0)
    _fill(ref, 1)
    for k in range(ROUNDS):
        ref.round(k)
    assert V_w == ref.V
    assert np.allclose(theta_w, ref.theta, rtol=0, atol=1e-15)
