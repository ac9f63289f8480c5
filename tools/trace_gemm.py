"""clock64 timeline of CTA (0,0,0) of each GEMM phase (needs GORILA_LIB=.../libgorila_trace.so)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GORILA_LIB", os.path.join(ROOT, "paper_1507_04296_b200", "libgorila_trace.so"))
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila, load  # noqa: E402

nA, B = 18, int(os.environ.get("B", "32"))
g = Gorila(n_actions=nA, batch=B, replay_capacity=5000, theta0=synth.theta0(nA), math="bf16")
f = synth.frames(synth.SEED_DATA, 0, 0, 5000)
a, r, d = synth.meta(synth.SEED_DATA, 0, 0, 5000, nA)
g.replay_insert(0, f, a, r, d)
ids = np.array([0], np.int32)
for k in range(3):
    g.round(ids, k)
names = {0: "entry", 1: "prologue", 2: "pdl_wait", 3: "producer_done", 4: "mma_done", 5: "epilogue_done",
         6: "dealloc", 16: "epi_row", 17: "ld0", 18: "st0", 19: "ld1", 20: "st1", 21: "ld2", 22: "st2", 23: "ld3",
         24: "st3"}
for ph in ["conv1_fwd", "conv2_fwd", "conv3_fwd", "fc4_fwd", "fc4_dgrad", "fc4_wgrad", "conv3_dgrad",
           "conv2_dgrad", "conv3_wgrad", "conv2_wgrad", "conv1_wgrad"]:
    us = g.bench_phase(ph, iters=50)
    g.bench_phase(ph, iters=1)
    buf = (ctypes.c_uint64 * 64)()
    load().gorila_debug_trace(buf)
    t = list(buf)
    t0 = t[0]
    ev = sorted([(v - t0, k) for k, v in enumerate(t) if v and v >= t0], key=lambda x: x[0])
    line = "  ".join(f"{names.get(k, 'issued%d' % (k - 8))}={v}" for v, k in ev if v < 10**7)
    print(f"{ph:12s} {us:6.2f} us/launch | {line}")
    if os.environ.get("RAW"):
        print("   raw:", [(k, v - t0) for k, v in enumerate(t) if v])
