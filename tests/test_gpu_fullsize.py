"""Parity at BASELINE.json's full single-GPU size, in the launch configuration bench.py times
(SURVEY §8(c) "C2: steps 0-9, 99-101 (around a sync)"; the C2 teacher-forced subset).

C2: nA = 18, B = 32, a 1,000,000-frame device replay filled by the device generator (the bench's
fill), rounds run through gorila_round (CUDA-graph replay), target sync every 100 versions. The
oracle cannot hold 7 GB of frames, but every frame and transition is a pure function of its slot
(synth, pinned device == host by test_gpu_parity::test_device_synth_matches_host), so for each
checked round the oracle rebuilds exactly the windows the round samples: indices from its own
Philox mapping (O2), the five frames tau-3 .. tau+1 and their transitions into a small oracle Ring,
stacked by the oracle's own gather (O3). It then runs O4-O12 from the GPU's state before the round
(teacher forcing): Q / Q-hat / loss, the outlier / sync decisions, G per tensor, the RMSProp step.
"""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_util import TOL, gpu_acts, per_tensor_rel_l2, rel_inf, rel_l2, replica_of, teacher_forced_acts

pytestmark = pytest.mark.gpu

NA, B, C, PERIOD = 18, 32, 1_000_000, 100
LR, RHO, EPS, GAMMA = 2.5e-4, 0.95, 0.01, 0.99


def _fill_device(g, nA, capacity, chunk=131072):
    import torch
    fr = torch.empty((chunk, 84, 84), dtype=torch.uint8, device="cuda")
    a = torch.empty(chunk, dtype=torch.uint8, device="cuda")
    r = torch.empty(chunk, dtype=torch.float32, device="cuda")
    d = torch.empty(chunk, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    t = 0
    while t < capacity:
        n = min(chunk, capacity - t)
        synth.fill_frames_dev(synth.SEED_DATA, 0, t, n, fr.data_ptr(), st)
        synth.fill_meta_dev(synth.SEED_DATA, 0, t, n, nA, 0.0, a.data_ptr(), r.data_ptr(), d.data_ptr(), st)
        g.replay_insert(0, fr[:n], a[:n], r[:n], d[:n])
        t += n
    torch.cuda.synchronize()


def _oracle_batch(tau):
    """s, s', a, r, d of the sampled slots, through the oracle's own ring and stacking (O3)."""
    S, S2 = np.zeros((B, 4, 84, 84), np.uint8), np.zeros((B, 4, 84, 84), np.uint8)
    A, R, D = np.zeros(B, np.uint8), np.zeros(B, np.float32), np.zeros(B, np.uint8)
    for i, t in enumerate(tau):
        lo = max(0, int(t) - 3)
        cnt = int(t) + 2 - lo
        ring = O.Ring(8)
        f = synth.frames(synth.SEED_DATA, 0, lo, cnt)
        a, r, d = synth.meta(synth.SEED_DATA, 0, lo, cnt, NA)
        ring.insert(f, a, r, d)
        s, s2, aa, rr, dd = ring.gather(np.array([int(t) - lo], np.int64))
        S[i], S2[i], A[i], R[i], D[i] = s[0], s2[0], aa[0], rr[0], dd[0]
    return S, S2, A, R, D


@pytest.mark.parametrize("math,check", [("bf16", (0, 1, 2, 98, 99, 100, 101)), ("fp32", (0, 1))])
def test_c2_full_size_sampled_parity(math, check):
    from paper_1507_04296_b200 import Gorila
    mode = "bf16" if math == "bf16" else "exact"
    tol = TOL[math]
    g = Gorila(n_actions=NA, batch=B, replay_capacity=C, theta0=synth.theta0(NA), math=math,
               target_period=PERIOD, history=2)
    _fill_device(g, NA, C)
    ids = np.array([0], np.int32)
    n_checked = 0
    forced = []  # teacher-forced ReLU decisions per checked round and layer (R30)
    for k in range(max(check) + 1):
        if k not in check:
            g.round(ids, k)
            continue
        th0, m0, v0, V0 = g.get_state()
        tm0, st0 = g.get_learner_state(0)
        gpu_s = g.replay_sample(0, k)
        info, rinfo, synced = g.round(ids, k, want_info=True)
        G = g.get_grad()
        q, qh = g.get_q(0)
        th1, _, _, V1 = g.get_state()
        tm1, st1 = g.get_learner_state(0)
        info = info[0]

        # O2 / O3: indices and gathered windows, bit-exact
        tau = O.sample_indices(C, C, B, 1507, 0, k)
        assert np.array_equal(gpu_s["tau"], tau)
        s, s2, a, r, d = _oracle_batch(tau)
        assert np.array_equal(gpu_s["s"], s) and np.array_equal(gpu_s["s2"], s2)
        assert np.array_equal(gpu_s["a"], a) and np.array_equal(gpu_s["r"], r) and np.array_equal(gpu_s["d"], d)

        # O4 - O6 from the GPU's parameters before the round
        Q, acts, zs = O.qnet_forward(th0, s, NA, mode, want_z=True)
        Qh, _ = O.qnet_forward(tm0, s2, NA, mode)
        assert rel_inf(q, Q) <= tol["q"] and rel_inf(qh, Qh) <= tol["q"], (k, rel_inf(q, Q), rel_inf(qh, Qh))
        _, _, dQ, loss, ell = O.td_terms(Q, Qh, a, r, d, GAMMA)
        assert abs(info["loss"] - loss) <= tol["loss"] * abs(loss)
        assert abs(info["abs_loss"] - ell) <= tol["loss"] * abs(ell)

        # O7 / O9: decisions (outlier exact outside the R9 margin; staleness off)
        stats = O.LossStats(mu=st0["mu"], var=st0["var"], count=st0["count"])
        thr = stats.mu + 3.0 * np.sqrt(stats.var)
        rejected = stats.rejects(ell, 3.0, 100)
        if stats.count < 100 or abs(ell - thr) > 1e-2 * abs(thr):
            assert bool(info["rejected_outlier"]) == bool(rejected)
        accepted = bool(info["accepted"])
        assert accepted == (not bool(info["rejected_outlier"]))
        assert rinfo["n_accepted"] == int(accepted) and V1 == V0 + int(accepted)

        # O8: gradient per tensor, the oracle's backward teacher-forced to the GPU's ambiguous ReLU
        # decisions (R30; gpu_acts = the round's learner activations, read after the graph round)
        if accepted:
            acts_tf = teacher_forced_acts(gpu_acts(g), acts, zs, math, forced)
            G_ref = O.qnet_backward(th0, s, acts_tf, dQ, NA, mode)
            assert rel_l2(G, G_ref) <= tol["g"], (k, "G", rel_l2(G, G_ref), forced[-1])
            for name, e in per_tensor_rel_l2(G, G_ref, NA).items():
                assert e <= tol["g"], (k, "G", name, e, forced[-1])
            # O10: the RMSProp step from the GPU's optimizer state, every tensor (+ fp32 state floor R31)
            th_ref, m_ref, v_ref = th0.astype(np.float64), m0.astype(np.float64), v0.astype(np.float64)
            O.rmsprop_apply(th_ref, m_ref, v_ref, G_ref, LR, RHO, EPS)
            d_gpu = th1.astype(np.float64) - th0
            th1_ref = th_ref.astype(np.float32)
            d_ref = th1_ref.astype(np.float64) - th0
            ulp = np.spacing(np.abs(th1_ref)).astype(np.float64)
            off = 0
            for name, shp in O.param_shapes(NA):
                n = int(np.prod(shp))
                sl = slice(off, off + n)
                if np.any(d_ref[sl]):
                    e = rel_l2(d_gpu[sl], d_ref[sl])
                    floor = np.linalg.norm(ulp[sl]) / np.linalg.norm(d_ref[sl])
                    assert e <= tol["dtheta"] + floor, (k, "dtheta", name, e, floor)
                off += n
        else:
            assert np.array_equal(th1, th0)

        # O12: target sync, integer-exact, and theta^- = the new replica when it fires
        want_sync = V1 >= st0["last_sync"] + PERIOD
        assert bool(synced[0]) == want_sync and st1["last_sync"] == (V1 if want_sync else st0["last_sync"])
        if want_sync:
            assert np.array_equal(tm1.astype(np.float64), replica_of(th1, NA, math))
        else:
            assert np.array_equal(tm1, tm0)
        n_checked += 1
    assert n_checked == len(check)
    g.close()
