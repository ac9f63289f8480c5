"""e2e loop variants (spin wait, lag 1): which per-step stream operations cost device time."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila  # noqa: E402

nA, C = 18, 200_000
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
g = Gorila(n_actions=nA, batch=32, replay_capacity=C, theta0=synth.theta0(nA), math="bf16", stream=stream)
f = synth.frames(synth.SEED_DATA, 0, 0, 20000)
a, r, d = synth.meta(synth.SEED_DATA, 0, 0, 20000, nA)
g.replay_insert(0, f, a, r, d)
ids = np.array([0], np.int32)
k = 0
for k in range(10):
    g.round(ids, k)
k += 1
f1 = torch.empty((1, 84, 84), dtype=torch.uint8).pin_memory()
a1 = torch.zeros(1, dtype=torch.uint8).pin_memory()
r1 = torch.zeros(1, dtype=torch.float32).pin_memory()
d1 = torch.zeros(1, dtype=torch.uint8).pin_memory()
N = 2000
for name, ins, res in (("round only", False, False), ("post, no fetch", False, None),
                       ("round+results", False, True), ("insert+round", True, False),
                       ("insert+round+results", True, True)):
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pend = None
    for i in range(N):
        if ins:
            g.replay_insert(0, f1, a1, r1, d1)
        if res is None:
            g.round_async(ids, k)
        elif res:
            h = g.round_async(ids, k)
            if pend is not None:
                g.round_result(pend)
            pend = h
        else:
            g.round(ids, k)
        k += 1
    if pend is not None:
        g.round_result(pend)
    e1.record(stream)
    stream.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name:22s} {ms / N * 1e3:6.1f} us/step  {N / ms * 1e3:7.0f} updates/s", flush=True)
