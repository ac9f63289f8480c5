"""e2e loop variants: result lag depth (round_async / round_result = gorila_round_post / _fetch)."""
import os
import sys
import time

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
stream.synchronize()
f1 = torch.empty((1, 84, 84), dtype=torch.uint8).pin_memory()
a1 = torch.zeros(1, dtype=torch.uint8).pin_memory()
r1 = torch.zeros(1, dtype=torch.float32).pin_memory()
d1 = torch.zeros(1, dtype=torch.uint8).pin_memory()
N = 1000

for spin in (False,):
    for lag in (1, 2, 3):
        pend = []
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for i in range(N):
            f1.numpy()[0] = f[i]
            a1.numpy()[0], r1.numpy()[0], d1.numpy()[0] = a[i], r[i], d[i]
            g.replay_insert(0, f1, a1, r1, d1)
            pend.append(g.round_async(ids, k)); k += 1
            if len(pend) > lag:
                h = pend.pop(0)
                g.round_result(h)
        for h in pend:
            g.round_result(h)
        e1.record(stream)
        stream.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"spin={spin} lag={lag}: {N / ms * 1e3:.0f} updates/s ({ms / N * 1e3:.1f} us/step, wall {(time.perf_counter() - t0) / N * 1e6:.1f})")
