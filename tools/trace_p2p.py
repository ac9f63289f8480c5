"""Where the peer-memory exchange spends its time (trace build; run under torchrun, N GPUs):
per round, the apply's wait for every peer's 'gradient ready' flag, its work after that wait
(block 0's wait end -> last block done), and k_peer_wait's wait for every peer's 'done'.
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/trace_p2p.py"""
import ctypes
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GORILA_LIB", os.path.join(ROOT, "paper_1507_04296_b200", "libgorila_trace.so"))
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila, load, nccl_unique_id  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
obj = [nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
nA, B, C = 18, 32, 20000
stream = torch.cuda.Stream()
g = Gorila(n_actions=nA, batch=B, replay_capacity=C, learner_id_base=rank, rank=rank, world=world,
           nccl_unique_id=obj[0], stream=stream, theta0=synth.theta0(nA), math="bf16", history=2)
f = synth.frames(synth.SEED_DATA, rank, 0, C)
a, r, d = synth.meta(synth.SEED_DATA, rank, 0, C, nA)
g.replay_insert(0, f, a, r, d)
ids = np.array([0], np.int32)
for k in range(20):
    g.round(ids, k)
stream.synchronize()
buf = (ctypes.c_uint64 * 64)()
load().gorila_debug_trace(buf)
base = [buf[i] for i in (40, 41, 42, 43)]
n = int(os.environ.get("ROUNDS", "500"))
for k in range(20, 20 + n):
    g.round(ids, k)
stream.synchronize()
load().gorila_debug_trace(buf)
cur = [buf[i] for i in (40, 41, 42, 43)]
dlt = [c - b for c, b in zip(cur, base)]
rounds = max(dlt[3], 1)
line = (f"[rank {rank}] rounds {dlt[3]}: apply wait-for-peers {dlt[0] / rounds / 1e3:.2f} us, apply work "
        f"{dlt[1] / rounds / 1e3:.2f} us, peer-done wait {dlt[2] / rounds / 1e3:.2f} us")
out = [None] * world
dist.all_gather_object(out, line)
if rank == 0:
    print("\n".join(out), flush=True)
g.close()
dist.destroy_process_group()
