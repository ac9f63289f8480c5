"""Quick A/B of the device-timed round (no e2e, no profile): prints one line per run.
usage: python tools/qbench.py [--batch B] [--steps K] [--capacity C] [--reps R]   (env knobs apply)"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--steps", type=int, default=3000)
ap.add_argument("--capacity", type=int, default=200_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--math", default="bf16")
ap.add_argument("--phases", default="", help="comma list of phases to time in isolation (gorila_bench_phase)")
a = ap.parse_args()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
g = Gorila(n_actions=18, batch=a.batch, replay_capacity=a.capacity, theta0=synth.theta0(18), math=a.math, stream=st)
bench.fill_replay(g, 0, a.capacity, 18, synth.SEED_DATA, 0)
ids = np.zeros(1, np.int32)
k = 0
for _ in range(20):
    g.round(ids, k)
    k += 1
res = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.synchronize()
    e0.record(st)
    for _ in range(a.steps):
        g.round(ids, k)
        k += 1
    e1.record(st)
    st.synchronize()
    res.append(e0.elapsed_time(e1) * 1000 / a.steps)
knobs = {k_: v for k_, v in os.environ.items() if k_.startswith("GORILA_")}
ap_us = g.bench_phase("apply", iters=200)
tw_us = g.bench_phase("conv1_fwd", iters=200)
print(f"B={a.batch} us/step {min(res):.2f} (reps {' '.join(f'{r:.2f}' for r in res)}) "
      f"updates/s {1e6 / min(res):.0f} apply(iso) {ap_us:.2f} us tower(iso) {tw_us:.2f} us knobs {knobs}", flush=True)
if a.phases:
    print({ph: round(g.bench_phase(ph, iters=50), 2) for ph in a.phases.split(",")}, flush=True)
g.close()
