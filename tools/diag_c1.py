"""Per-round parity diagnostics for the C1 teacher-forced run (prints every error metric)."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_util import make_pair, teacher_force, run_round_both, per_tensor_rel_l2, rel_inf, rel_l2
math = sys.argv[1] if len(sys.argv) > 1 else "fp32"
g, orc = make_pair(nA=4, B=32, C=10_000, n_insert=10_000, math=math, target_period=5, outlier_warmup=2)
for k in range(10):
    teacher_force(g, orc)
    gpu, res = run_round_both(g, orc, k, [0])
    oi = res["learners"][0]
    q, qh = gpu["q"][0]
    Gref = oi.get("G", np.zeros(1))
    print(k, "acc", gpu["info"][0]["accepted"], oi["accepted"], "rej", gpu["info"][0]["rejected_outlier"],
          "Q %.1e Qh %.1e" % (rel_inf(q, oi["Q"]), rel_inf(qh, oi["Qhat"])),
          "G %.1e" % rel_l2(gpu["G"], Gref) if oi["accepted"] else "",
          {k2: "%.1e" % v for k2, v in per_tensor_rel_l2(gpu["G"], Gref, 4).items()} if oi["accepted"] else "",
          "synced", gpu["synced"][0], res["synced"][0], "max|delta|", np.abs(oi["delta"]).max())
