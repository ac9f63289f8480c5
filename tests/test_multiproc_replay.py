"""world_size-2 gloo test (CPU) of the global-replay protocol (NEXT row f4; R36).

Each process is one rank holding only its own learner's ring, as on the GPUs. Per round, as the
library does it over NVLink: the replay barrier publishes every rank's ring counter (here: an
all-gather), each rank draws its learner's (shard, tau) over the union in rank-major shard order,
and fetches the windows of the samples that fall in a peer's ring from that peer (here: request
lists and stacked windows exchanged with all_gather_object; on the GPUs the sampler reads the
peer's HBM). Between rounds the ranks insert different amounts of new experience. Every rank's
batch -- shard, tau, s, s', a, r, d -- must equal the single-process oracle's global draw with
both learners' rings in one place.
"""
import os

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth

NA, B, C, ROUNDS, W = 4, 16, 400, 4, 2
FILL = {0: 500, 1: 150}           # initial steps per rank (rank 0's ring wraps)
MORE = {0: (7, 0, 3), 1: (0, 40, 1)}  # steps inserted before rounds 1, 2, 3


def _insert(ring, j, t0, n):
    if n:
        ring.insert(synth.frames(synth.SEED_DATA, j, t0, n), *synth.meta(synth.SEED_DATA, j, t0, n, NA))


def _rank_main(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    ring = O.Ring(C)
    _insert(ring, rank, 0, FILL[rank])
    t = FILL[rank]
    batches = []
    for k in range(ROUNDS):
        if k:
            _insert(ring, rank, t, MORE[rank][k - 1])
            t += MORE[rank][k - 1]
        # replay barrier: every rank's counter, as of the round's start
        ns = [None] * W
        dist.all_gather_object(ns, ring.n)
        shard, tau = O.sample_indices_global(ns, C, B, 1507, rank, k)
        # requests to each shard's owner; owners answer with their stacked windows
        reqs = [None] * W
        dist.all_gather_object(reqs, {q: tau[shard == q].tolist() for q in range(W)})
        mine = {q: ring.gather(np.array(reqs[q][rank], np.int64)) if reqs[q][rank] else None for q in range(W)}
        answers = [None] * W
        dist.all_gather_object(answers, mine)
        parts = [np.zeros((B, 4, 84, 84), np.uint8), np.zeros((B, 4, 84, 84), np.uint8),
                 np.zeros(B, np.uint8), np.zeros(B, np.float32), np.zeros(B, np.uint8)]
        for q in range(W):
            sel = np.nonzero(shard == q)[0]
            if len(sel):
                got = answers[q][rank]
                for f in range(5):
                    parts[f][sel] = got[f]
        batches.append((shard, tau, *parts))
    out.put((rank, batches))
    dist.destroy_process_group()


def test_global_replay_across_ranks_equals_single_process_union():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + 7
    procs = [ctx.Process(target=_rank_main, args=(r, port, out)) for r in range(W)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=600) for _ in range(W))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rings = [O.Ring(C) for _ in range(W)]
    t = dict(FILL)
    for j in range(W):
        _insert(rings[j], j, 0, FILL[j])
    seen = set()
    for k in range(ROUNDS):
        if k:
            for j in range(W):
                _insert(rings[j], j, t[j], MORE[j][k - 1])
                t[j] += MORE[j][k - 1]
        for j in range(W):
            shard, tau = O.sample_indices_global([rg.n for rg in rings], C, B, 1507, j, k)
            ref = (shard, tau, *O.gather_global(rings, shard, tau))
            for x, y in zip(got[j][k], ref):
                assert np.array_equal(x, y)
            seen |= set(shard.tolist())
    assert seen == {0, 1}
