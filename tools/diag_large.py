"""Diagnostics of the large-batch parity (tests/test_gpu_large_batch.py's construction): per-tensor G
errors and, layer by layer, how many bf16 output-gradient elements (g4..g1) differ between the GPU
and the oracle's own backward (teacher-forced activations), with the size of the differences."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from gpu_util import (gpu_acts, make_pair, per_tensor_rel_l2, round_bf16_vec, teacher_force,  # noqa: E402
                      teacher_forced_acts)


def run(B, math, nA=18, C=64):
    g, orc = make_pair(nA=nA, B=B, C=C, n_insert=C, math=math, outlier_enabled=False)
    teacher_force(g, orc)
    mode = "bf16" if math == "bf16" else "exact"
    th0 = g.get_state()[0]
    tm0, _ = g.get_learner_state(0)
    g.capture_activations(True)
    g.learner_step([0], 0)
    G = g.get_grad()
    ring = orc.learners[0].ring
    tau = O.sample_indices(ring.n, ring.size, B, 1507, 0, 0)
    uniq, first, inv, cnt = np.unique(tau, return_index=True, return_inverse=True, return_counts=True)
    s, s2, a, r, d = ring.gather(uniq)
    Q, acts, zs = O.qnet_forward(th0, s, nA, mode, want_z=True)
    Qh, _ = O.qnet_forward(tm0, s2, nA, mode)
    _, delta, _, _, _ = O.td_terms(Q, Qh, a, r, d, 0.99)
    dQ = np.zeros_like(Q)
    dQ[np.arange(len(uniq)), a.astype(int)] = -np.clip(delta, -1.0, 1.0) / B
    forced = []
    acts_tf = teacher_forced_acts(gpu_acts(g, 0, rows=first), acts, zs, math, forced)
    G_ref = sum(cnt[u] * O.qnet_backward(th0, s[u:u + 1], acts_tf[u:u + 1], dQ[u:u + 1], nA, mode)
                for u in range(len(uniq)))
    errs = per_tensor_rel_l2(G, G_ref, nA)
    print(f"B={B} {math} unique={len(uniq)} forced={forced} " + " ".join(f"{k}:{v:.2e}" for k, v in errs.items()),
          flush=True)
    if math != "bf16":
        return
    # the oracle's output gradients, layer by layer (oracle.c backward, BF16 mode, dQ per distinct stack
    # scaled by its count: the GPU's per-sample g is dQ_b-scaled, so compare g / cnt)
    p = O.unflatten(th0, nA)
    q = round_bf16_vec
    n1, n2, n3 = 12800, 5184, 3136
    a1 = acts_tf[:, :n1].reshape(-1, 32, 20, 20)
    a2 = acts_tf[:, n1:n1 + n2].reshape(-1, 64, 9, 9)
    a3 = acts_tf[:, n1 + n2:n1 + n2 + n3]
    a4 = acts_tf[:, n1 + n2 + n3:]
    dq1 = dQ
    g4 = q(np.where(a4 > 0, O.linear_bwd_data(dq1, p["W5"]), 0.0))
    g3 = q(np.where(a3 > 0, O.linear_bwd_data(g4, q(p["W4"])), 0.0))
    g2 = q(np.where(a2 > 0, O.conv2d_bwd_data(g3.reshape(-1, 64, 7, 7), q(p["W3"]), (9, 9), 1), 0.0))
    g1 = q(np.where(a1 > 0, O.conv2d_bwd_data(g2, q(p["W2"]), (20, 20), 2), 0.0))
    for name, ref, shp in (("g4", g4, (512,)), ("g3", g3, (7, 7, 64)), ("g2", g2, (9, 9, 64)), ("g1", g1, (20, 20, 32))):
        x = g.get_activation(name).reshape((B,) + shp)[first]
        if len(shp) == 3:
            x = x.transpose(0, 3, 1, 2)
        x = x.reshape(len(first), -1).astype(np.float64)
        ref = ref.reshape(len(first), -1)
        diff = x != ref
        scale = np.abs(ref).max()
        rel = np.abs(x - ref)[diff] / np.maximum(np.abs(ref[diff]), 1e-30) if diff.any() else np.zeros(1)
        print(f"   {name}: differ at {diff.sum()} of {diff.size} ({diff.mean():.2e}); median rel diff {np.median(rel):.2e} "
              f"max |diff|/max|ref| {np.abs(x - ref).max() / scale:.2e}; l2 rel {np.linalg.norm(x - ref) / np.linalg.norm(ref):.2e}",
              flush=True)
    g.close()


for B in (32, 300, 1024, 4096):
    run(B, "bf16")
run(1024, "fp32")
