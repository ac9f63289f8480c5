"""Pins of the oracle's global replay draw (NEXT row f4; reading R36).

D = the union of the shards' valid transitions ("a global replay memory aggregates the experience
into a distributed database", §4; minibatches "sampled from either a local or global
experience replay memory D"), sampled uniformly (§3.3). Pinned against: the explicit
enumeration of the union with an independent Philox and big-int arithmetic (brute force), the
single-shard special case (= the local draw O2, itself pinned in test_oracle_primitives), the
shard proportions and within-shard uniformity (chi-square), empty shards, and a whole round
that must equal the local-replay round when the other shards hold no valid transition.
"""
import numpy as np
import pytest

import oracle as O
import synth


def _u(seed, learner, rnd, i):
    key = [seed & 0xFFFFFFFF, seed >> 32]
    x = synth.philox([i // 2, learner, rnd & 0xFFFFFFFF, ((rnd >> 32) & 0xFFFFFF) | (3 << 24)], key)
    return int(x[0]) | (int(x[1]) << 32) if i % 2 == 0 else int(x[2]) | (int(x[3]) << 32)


@pytest.mark.parametrize("ns,C", [([5, 1, 9, 30], 12), ([2, 2], 100), ([0, 40, 3], 16), ([100, 7], 50)])
def test_global_draw_is_the_indexed_union(ns, C):
    # brute force: list D explicitly (shard order, then tau ascending), index it with floor(u*|D|/2^64)
    union = []
    for j, n in enumerate(ns):
        size = min(n, C)
        union += [(j, t) for t in range(n - size, n - 1)]  # valid tau: [n - size, n - 2]
    seed, learner, rnd, B = 1507, 2, (1 << 32) + 5, 37
    shard, tau = O.sample_indices_global(ns, C, B, seed, learner, rnd)
    for i in range(B):
        j, t = union[_u(seed, learner, rnd, i) * len(union) >> 64]
        assert (shard[i], tau[i]) == (j, t)


@pytest.mark.parametrize("n,C", [(10, 10), (1000, 64), (2, 2), (123_456, 100_000)])
def test_single_shard_is_the_local_draw(n, C):
    for rnd in (0, 7, (1 << 33) + 1):
        shard, tau = O.sample_indices_global([n], C, 32, 1507, 3, rnd)
        assert (shard == 0).all()
        assert np.array_equal(tau, O.sample_indices(n, min(n, C), 32, 1507, 3, rnd))


def test_empty_shards_are_never_drawn_and_all_empty_is_not_ready():
    for rnd in range(30):
        shard, tau = O.sample_indices_global([1, 50, 0, 1, 20], 64, 64, 9, 0, rnd)
        assert set(shard.tolist()) <= {1, 4}
    with pytest.raises(ValueError):
        O.sample_indices_global([1, 0, 1], 8, 4, 1, 0, 0)


def test_shard_proportions_and_within_shard_uniformity():
    # P(shard j) = (size_j - 1) / sum (size - 1); uniform within the shard's valid slots
    from scipy.stats import chisquare
    ns, C = [41, 201, 1001, 1], 600
    M = np.array([min(n, C) - 1 if min(n, C) >= 2 else 0 for n in ns], np.float64)
    draws = [O.sample_indices_global(ns, C, 1000, 1507, 1, k) for k in range(150)]
    shard = np.concatenate([d[0] for d in draws])
    tau = np.concatenate([d[1] for d in draws])
    hist = np.bincount(shard, minlength=len(ns))
    assert hist[3] == 0
    exp = M[:3] / M.sum() * shard.size
    assert chisquare(hist[:3], exp).pvalue > 0.01
    for j in (1, 2):  # within-shard uniformity over [n - size, n - 2]
        size = min(ns[j], C)
        h = np.bincount(tau[shard == j] - (ns[j] - size), minlength=size - 1)
        assert h.size == size - 1 and chisquare(h).pvalue > 0.001


def _oracle(replay_mode):
    cfg = O.Config(n_actions=4, batch=8, capacity=64, learners=(0, 1), mode="exact", outlier_enabled=False,
                   replay_mode=replay_mode)
    o = O.GorilaOracle(cfg, synth.theta0(4))
    f = synth.frames(synth.SEED_DATA, 0, 0, 40)
    a, r, d = synth.meta(synth.SEED_DATA, 0, 0, 40, 4)
    o.insert(0, f, a, r, d)
    f1 = synth.frames(synth.SEED_DATA, 1, 0, 1)
    a1, r1, d1 = synth.meta(synth.SEED_DATA, 1, 0, 1, 4)
    o.insert(1, f1, a1, r1, d1)  # one step: no valid transition yet (not ready)
    return o


def test_global_round_equals_local_round_when_other_shards_are_empty():
    lo, gl = _oracle("local"), _oracle("global")
    for k in range(3):
        pl, pg = lo.round(k)["learners"], gl.round(k)["learners"]
        assert pl[1]["not_ready"] and pg[1]["not_ready"]
        assert np.array_equal(pl[0]["tau"], pg[0]["tau"]) and (pg[0]["shard"] == 0).all()
    assert np.array_equal(lo.theta, gl.theta)


def test_global_round_gathers_from_the_drawn_shard():
    o = _oracle("global")
    f1 = synth.frames(synth.SEED_DATA, 1, 1, 30)
    a1, r1, d1 = synth.meta(synth.SEED_DATA, 1, 1, 30, 4)
    o.insert(1, f1, a1, r1, d1)
    rings = [o.learners[0].ring, o.learners[1].ring]
    seen = set()
    for k in range(4):
        per = o.round(k)["learners"]
        for j in (0, 1):
            sh, tau = per[j]["shard"], per[j]["tau"]
            seen |= set(sh.tolist())
            for i in range(len(tau)):  # a, r, d of sample i are those of (shard, tau) in that ring
                s, s2, a, r, d = rings[sh[i]].gather(np.array([tau[i]]))
                assert (per[j]["a"][i], per[j]["r"][i], per[j]["d"][i]) == (a[0], r[0], d[0])
    assert seen == {0, 1}
