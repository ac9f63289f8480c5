"""NEXT row f3 measurement: batched epsilon-greedy acting throughput on 1 GPU (device-resident
states, wall-clocked around synchronous gorila_act calls, which include the action / Q read-back).
usage: python tools/bench_act.py [n_states] [iters]  -> one JSON line"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
nA = 18
g = Gorila(n_actions=nA, batch=n, replay_capacity=5000, theta0=synth.theta0(nA), math="bf16")
f = synth.frames(synth.SEED_DATA, 0, 0, 5000)
a, r, d = synth.meta(synth.SEED_DATA, 0, 0, 5000, nA)
g.replay_insert(0, f, a, r, d)
states = torch.from_numpy(g.replay_sample(0, 0)["s"]).cuda()
for k in range(20):
    g.act(states, k)
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(iters):
    g.act(states, 20 + k)
t1 = time.perf_counter()
print(json.dumps({"metric": "epsilon-greedy actions/s (batched acting, NEXT row f3)", "value": iters * n / (t1 - t0),
                  "unit": "actions/s", "n_states_per_call": n, "us_per_call": (t1 - t0) / iters * 1e6,
                  "timing": "host wall clock around synchronous calls (device-resident states; includes the "
                            "action and Q read-back)", "math": "bf16", "n_actions": nA}))
