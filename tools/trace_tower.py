"""clock64 timeline of CTA (0, 0) of the conv tower (trace build), one bench_phase launch."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GORILA_LIB", os.path.join(ROOT, "paper_1507_04296_b200", "libgorila_trace.so"))
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila, load  # noqa: E402

g = Gorila(n_actions=18, batch=32, replay_capacity=5000, theta0=synth.theta0(18), math="bf16")
f = synth.frames(synth.SEED_DATA, 0, 0, 5000)
a, r, d = synth.meta(synth.SEED_DATA, 0, 0, 5000, 18)
g.replay_insert(0, f, a, r, d)
ids = np.array([0], np.int32)
for k in range(3):
    g.round(ids, k)
print("conv1_fwd (tower) isolated us:", g.bench_phase("conv1_fwd", iters=50))
g.bench_phase("conv1_fwd", iters=1)
buf = (ctypes.c_uint64 * 64)()
load().gorila_debug_trace(buf)
names = {48: "start(after pdl)", 49: "s planes landed", 50: "conv1 MMAs issued", 51: "a1 in smem (mma)",
         52: "conv2 MMAs issued", 53: "a2 in smem (mma)", 54: "conv3 MMAs issued", 55: "conv1 acc ready (epi)",
         56: "a1 written (epi)", 57: "conv2 acc ready (epi)", 58: "a2 written (epi)", 59: "conv3 acc ready (epi)",
         60: "end"}
t0 = buf[48]
for sl in sorted(names, key=lambda s: buf[s]):
    print(f"{names[sl]:24s} {int(buf[sl]) - int(t0):8d} cycles")
