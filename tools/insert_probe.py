"""Where the e2e replay_insert host time goes: insert / bare H2D copy / bare launch, idle vs busy stream."""
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
for k in range(10):
    g.round(ids, k)
stream.synchronize()
f1 = torch.empty((1, 84, 84), dtype=torch.uint8).pin_memory()
a1 = torch.zeros(1, dtype=torch.uint8).pin_memory()
r1 = torch.zeros(1, dtype=torch.float32).pin_memory()
d1 = torch.zeros(1, dtype=torch.uint8).pin_memory()
hbuf = torch.zeros(7062, dtype=torch.uint8).pin_memory()
dbuf = torch.zeros(7062, dtype=torch.uint8, device="cuda")
x = torch.zeros(1, device="cuda")
N = 300
k = 10


def timed(fn, busy):
    global k
    tot = 0.0
    for _ in range(N):
        if busy:
            g.round(ids, k)
            k += 1
        t0 = time.perf_counter()
        fn()
        tot += time.perf_counter() - t0
        stream.synchronize()
    return round(tot / N * 1e6, 1)


for busy in (False, True):
    print("busy" if busy else "idle",
          "insert", timed(lambda: g.replay_insert(0, f1, a1, r1, d1), busy),
          "h2d7k", timed(lambda: dbuf.copy_(hbuf, non_blocking=True), busy),
          "launch", timed(lambda: x.add_(1), busy),
          "round_async", timed(lambda: g.round_result(g.round_async(ids, 0)) if False else g.round_async(ids, k), busy))
