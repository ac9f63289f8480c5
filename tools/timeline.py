"""Per-kernel timeline of a few B=32 rounds (torch.profiler / CUPTI: concurrent kernels, graph
replays included): prints, for the last profiled round, each kernel's start and end relative to
the round's first kernel, its stream and duration. usage: python tools/timeline.py [--batch B]"""
import argparse
import json
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
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--out", default="gpurun_out/timeline.json")
a = ap.parse_args()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
g = Gorila(n_actions=18, batch=a.batch, replay_capacity=100_000, theta0=synth.theta0(18), stream=st)
bench.fill_replay(g, 0, 100_000, 18, synth.SEED_DATA, 0)
ids = np.zeros(1, np.int32)
k = 0
for _ in range(30):
    g.round(ids, k)
    k += 1
st.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.rounds):
        g.round(ids, k)
        k += 1
    st.synchronize()
prof.export_chrome_trace(a.out)
ev = [e for e in json.load(open(a.out))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
# rounds start at the sampler kernel
starts = [i for i, e in enumerate(ev) if "k_sample" in e["name"]]
i0 = starts[-2]
i1 = starts[-1]
t0 = ev[i0]["ts"]
print(f"round period {ev[i1]['ts'] - t0:.2f} us; kernels of one round:")
for e in ev[i0:i1]:
    nm = e["name"].split("(")[0].replace("void ", "")[:90]
    print(f"  {e['ts'] - t0:7.2f} -> {e['ts'] - t0 + e['dur']:7.2f}  ({e['dur']:6.2f})  s{e['args'].get('stream', '?')}  {nm}")
g.close()
