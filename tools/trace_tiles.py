"""Per-tile role timeline of CTA 0 of the shifted-window GEMMs (needs the trace build:
python -c 'from paper_1507_04296_b200 import _build; _build.build(trace=True)'), e.g.
B=4096 PH=conv1_fwd,conv2_dgrad python tools/trace_tiles.py"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GORILA_LIB", os.path.join(ROOT, "paper_1507_04296_b200", "libgorila_trace.so"))
import bench  # noqa: E402
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila, load  # noqa: E402

nA, B = 18, int(os.environ.get("B", "4096"))
g = Gorila(n_actions=nA, batch=B, replay_capacity=100000, theta0=synth.theta0(nA), math="bf16")
bench.fill_replay(g, 0, 100000, nA, synth.SEED_DATA, 0)
ids = np.array([0], np.int32)
for k in range(3):
    g.round(ids, k)
EV = ["cv_start", "cv_done", "mma_ops", "mma_acc", "mma_done", "ep_wait", "ep_ready", "ep_done"]
for ph in os.environ.get("PH", "conv1_fwd,conv2_dgrad").split(","):
    us = g.bench_phase(ph, iters=20)
    buf = (ctypes.c_uint64 * 512)()
    ctypes.memset(buf, 0, 8 * 512)
    g.bench_phase(ph, iters=1)
    load().gorila_debug_trace_tiles(buf)
    t = np.array(list(buf), np.int64).reshape(8, 64)
    t0 = t[t > 0].min() if (t > 0).any() else 0
    print(f"== {ph}: {us:.2f} us/launch (CTA 0, clock64 cycles from its first event)")
    print("tile " + " ".join(f"{e:>9s}" for e in EV))
    for tl in range(64):
        if not (t[:, tl] > 0).any():
            continue
        print(f"{tl:4d} " + " ".join(f"{(v - t0) if v else -1:9d}" for v in t[:, tl]))
