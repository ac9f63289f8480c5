"""Host-side cost per call of the e2e loop's pieces (wall clock, 1 GPU, configs[1] shapes)."""
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
N = 500
t = {"numpy fill": 0.0, "replay_insert": 0.0, "round_async": 0.0, "round_result": 0.0}
k = 10
pend = None
t_all0 = time.perf_counter()
for i in range(N):
    t0 = time.perf_counter()
    f1.numpy()[0] = f[i]
    a1.numpy()[0], r1.numpy()[0], d1.numpy()[0] = a[i], r[i], d[i]
    t1 = time.perf_counter()
    g.replay_insert(0, f1, a1, r1, d1)
    t2 = time.perf_counter()
    h = g.round_async(ids, k)
    t3 = time.perf_counter()
    if pend is not None:
        g.round_result(pend)
    t4 = time.perf_counter()
    pend = h
    k += 1
    t["numpy fill"] += t1 - t0
    t["replay_insert"] += t2 - t1
    t["round_async"] += t3 - t2
    t["round_result"] += t4 - t3
g.round_result(pend)
t_all = time.perf_counter() - t_all0
print({kk: round(v / N * 1e6, 1) for kk, v in t.items()}, "us per step; total", round(t_all / N * 1e6, 1))
t0 = time.perf_counter()
for i in range(N):
    g.round(ids, k)
    k += 1
stream.synchronize()
print("round (no info) back to back:", round((time.perf_counter() - t0) / N * 1e6, 1), "us per step")
# inserts alone (idle stream), then interleaved with asynchronous rounds
t0 = time.perf_counter()
for i in range(N):
    g.replay_insert(0, f1, a1, r1, d1)
stream.synchronize()
print("replay_insert back to back (idle stream):", round((time.perf_counter() - t0) / N * 1e6, 1), "us")
t0 = time.perf_counter()
ti = 0.0
for i in range(N):
    g.round(ids, k)
    k += 1
    s0 = time.perf_counter()
    g.replay_insert(0, f1, a1, r1, d1)
    ti += time.perf_counter() - s0
stream.synchronize()
print("insert while rounds are queued:", round(ti / N * 1e6, 1), "us; loop", round((time.perf_counter() - t0) / N * 1e6, 1))
