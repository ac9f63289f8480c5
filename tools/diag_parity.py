import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_util import make_pair, teacher_force, run_round_both, per_tensor_rel_l2, rel_inf, rel_l2
for math in ("fp32", "bf16"):
    for nA, B in ((4, 32), (18, 33)):
        g, orc = make_pair(nA=nA, B=B, C=5000, n_insert=5000, math=math, outlier_enabled=False)
        teacher_force(g, orc)
        gpu, res = run_round_both(g, orc, 0, [0])
        oi = res["learners"][0]; q, qh = gpu["q"][0]
        print(math, nA, B, "Q %.2e Qh %.2e loss %.2e" % (rel_inf(q, oi["Q"]), rel_inf(qh, oi["Qhat"]), abs(gpu["info"][0]["loss"]-oi["loss"])/oi["loss"]))
        print("   G", {k: "%.1e" % v for k, v in per_tensor_rel_l2(gpu["G"], oi["G"], nA).items()})
