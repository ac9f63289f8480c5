"""Parity at BASELINE configs[3]'s large per-GPU batches (B = 1024 and 4096), in the launch
configuration those batches use (persistent / shifted-window GEMMs, fc4 with M = samples, the
wide fc5 + TD kernel).

The oracle cannot run a 4096-sample forward / backward in a test, but the learner update is a
sum over samples: the replay here holds only 64 transitions, so the batch contains at most 63
distinct stacks, each drawn c_u times (O2's own index map). The oracle computes Q, Q-hat and the
TD terms of each distinct stack once, the loss as the multiplicity-weighted mean, and G as the
sum of the distinct stacks' per-sample gradients weighted by c_u (Eq.2 sums over the batch).
Every sample's Q / Q-hat is compared, G per tensor and the update per tensor at the full
tolerance, with the oracle's backward teacher-forced to the GPU's ambiguous ReLU decisions (R30).
"""
import numpy as np
import pytest

import oracle as O
from gpu_util import TOL, gpu_acts, make_pair, per_tensor_rel_l2, rel_inf, rel_l2, teacher_force, teacher_forced_acts

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("math", ["bf16", "fp32"])
@pytest.mark.parametrize("B", [1024, 4096])
def test_large_batch_update_parity(B, math):
    nA, C, gamma = 18, 64, 0.99
    g, orc = make_pair(nA=nA, B=B, C=C, n_insert=C, math=math, outlier_enabled=False)
    teacher_force(g, orc)
    mode = "bf16" if math == "bf16" else "exact"
    tol = TOL[math]
    th0, m0, v0, _ = g.get_state()
    tm0, _ = g.get_learner_state(0)
    g.capture_activations(True)
    info = g.learner_step([0], 0)[0]
    G = g.get_grad()
    q, qh = g.get_q(0)
    g.ps_apply_shard(0)
    th1 = g.get_state()[0]

    ring = orc.learners[0].ring
    tau = O.sample_indices(ring.n, ring.size, B, 1507, 0, 0)
    uniq, first, inv, cnt = np.unique(tau, return_index=True, return_inverse=True, return_counts=True)
    assert len(uniq) <= C - 1 and cnt.sum() == B
    s, s2, a, r, d = ring.gather(uniq)
    Q, acts, zs = O.qnet_forward(th0, s, nA, mode, want_z=True)
    Qh, _ = O.qnet_forward(tm0, s2, nA, mode)
    # every sample against its distinct stack
    assert rel_inf(q, Q[inv]) <= tol["q"] and rel_inf(qh, Qh[inv]) <= tol["q"], (rel_inf(q, Q[inv]), rel_inf(qh, Qh[inv]))
    y, delta, _, _, _ = O.td_terms(Q, Qh, a, r, d, gamma)
    loss = float(np.sum(cnt * delta ** 2) / B)
    assert abs(info["loss"] - loss) <= tol["loss"] * abs(loss)
    dQ = np.zeros_like(Q)
    dQ[np.arange(len(uniq)), a.astype(int)] = -np.clip(delta, -1.0, 1.0) / B
    forced = []
    acts_tf = teacher_forced_acts(gpu_acts(g, 0, rows=first), acts, zs, math, forced)
    # G = sum_u c_u G_u: one backward per distinct stack (in BF16 mode each sample's output gradients
    # are rounded per sample, R16, so the multiplicity scales the per-sample gradient, not dQ)
    G_ref = np.zeros(len(th0))
    for u in range(len(uniq)):
        G_ref += cnt[u] * O.qnet_backward(th0, s[u:u + 1], acts_tf[u:u + 1], dQ[u:u + 1], nA, mode)
    assert rel_l2(G, G_ref) <= tol["g"], (rel_l2(G, G_ref), forced)
    for name, e in per_tensor_rel_l2(G, G_ref, nA).items():
        assert e <= tol["g"], (name, e, forced)
    th_ref, m_ref, v_ref = th0.astype(np.float64), m0.astype(np.float64), v0.astype(np.float64)
    O.rmsprop_apply(th_ref, m_ref, v_ref, G_ref, 2.5e-4, 0.95, 0.01)
    d_gpu = th1.astype(np.float64) - th0
    th1_ref = th_ref.astype(np.float32)
    d_ref = th1_ref.astype(np.float64) - th0
    ulp = np.spacing(np.abs(th1_ref)).astype(np.float64)
    off = 0
    for name, shp in O.param_shapes(nA):
        n = int(np.prod(shp))
        sl = slice(off, off + n)
        off += n
        e = rel_l2(d_gpu[sl], d_ref[sl])
        floor = np.linalg.norm(ulp[sl]) / np.linalg.norm(d_ref[sl])
        assert e <= tol["dtheta"] + floor, ("dtheta", name, e, floor)
    g.close()


@pytest.mark.parametrize("B", [130, 300])
def test_ring_gather_descriptors_match_oracle_stacking(B):
    """B >= 75 (bf16): no stacked s is written; conv1 gathers its input from the replay ring through the
    sampler's per-sample descriptors (the five frame addresses and the episode / eviction keep bits,
    P:121 O3, DESIGN R3). The stack those descriptors describe (gorila_get_activation("s") expands it
    with the converters' gather) equals the oracle's O3 stacking bit for bit, on a wrapped ring with
    dense episode ends."""
    def dense_terms(j, d):
        d = d.copy()
        d[::5] = 1
        return d

    g, orc = make_pair(nA=6, B=B, C=500, n_insert=1337, math="bf16", terminals=dense_terms)
    ring = orc.learners[0].ring
    for k in (0, 3):
        g.round(np.array([0], np.int32), k)
        s_gpu = g.get_activation("s")  # [B][84][84][4], bf16 widened (integers: exact)
        tau = O.sample_indices(ring.n, ring.size, B, 1507, 0, k)
        s = ring.gather(tau)[0]  # [B][4][84][84] u8
        assert np.array_equal(s_gpu.transpose(0, 3, 1, 2), s.astype(np.float32)), k
    g.close()
