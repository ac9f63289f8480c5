"""Run the C1 bf16 teacher-forced rounds with two GORILA_SHIFT masks side by side and report, for
round K, where the intermediate tensors of the two GPU paths first differ (diagnostics).
usage: python tools/diag_modes.py K maskA maskB"""
import os
import sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_util import make_pair, teacher_force, run_round_both, per_tensor_rel_l2

K, ma, mb = int(sys.argv[1]), sys.argv[2], sys.argv[3]
pairs = []
for m in (ma, mb):
    os.environ["GORILA_SHIFT"] = m
    pairs.append(make_pair(nA=4, B=32, C=10_000, n_insert=10_000, math="bf16", target_period=5, outlier_warmup=2))
for k in range(K + 1):
    outs = []
    for g, orc in pairs:
        teacher_force(g, orc)
        outs.append(run_round_both(g, orc, k, [0]))
(gA, oA), (gB, oB) = pairs
for n in ("s", "a1", "a2", "a3", "a4", "g4", "g3", "g2", "g1"):
    x, y = gA.get_activation(n), gB.get_activation(n)
    d = np.abs(x - y)
    print(f"{n}: differing elements {int((d > 0).sum())} of {x.size}, max |diff| {d.max():.3e}, "
          f"max |x| {np.abs(x).max():.3e}")
    if 0 < (d > 0).sum() <= 5:
        for i in np.argwhere(d > 0):
            print("    ", tuple(int(v) for v in i), x[tuple(i)], y[tuple(i)])
GA, GB = outs[0][0]["G"], outs[1][0]["G"]
Gref = outs[0][1]["learners"][0].get("G")
print("G(A) vs ref", {k2: f"{v:.1e}" for k2, v in per_tensor_rel_l2(GA, Gref, 4).items()})
print("G(B) vs ref", {k2: f"{v:.1e}" for k2, v in per_tensor_rel_l2(GB, Gref, 4).items()})
