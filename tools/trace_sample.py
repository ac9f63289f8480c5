"""Sampler timeline in global-replay mode (trace build, torchrun, 2+ ranks): clock64 cycles per
block between: start -> shard counters read -> (shard, tau) -> flags in smem -> end, split by
whether the drawn shard is this rank's ring or a peer's."""
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

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
obj = [nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
C = int(os.environ.get("CAP", "200000"))
g = Gorila(n_actions=18, batch=32, replay_capacity=C, learner_id_base=rank, rank=rank, world=world,
           nccl_unique_id=obj[0], theta0=synth.theta0(18), math="bf16", replay_mode="global")
f = synth.frames(synth.SEED_DATA, rank, 0, 20000)
a, r, d = synth.meta(synth.SEED_DATA, rank, 0, 20000, 18)
g.replay_insert(0, f, a, r, d)
ids = np.array([0], np.int32)
for k in range(5):
    g.round(ids, k)
torch.cuda.synchronize()
buf0 = (ctypes.c_uint64 * 64)()
buf1 = (ctypes.c_uint64 * 64)()
load().gorila_debug_trace(buf0)
us = g.bench_phase("sample", iters=100)
torch.cuda.synchronize()
load().gorila_debug_trace(buf1)
dlt = [int(buf1[i]) - int(buf0[i]) for i in range(16)]
for o, name in ((0, "own shard"), (8, "peer shard")):
    n = max(dlt[o + 4], 1)
    print(f"[rank {rank}] sample {us:.1f} us; {name}: {dlt[o + 4]} blocks; mean cycles: counters {dlt[o] / n:.0f}, "
          f"draw {dlt[o + 1] / n:.0f}, flags {dlt[o + 2] / n:.0f}, frames+stores {dlt[o + 3] / n:.0f}", flush=True)
dist.barrier()
g.close()
dist.destroy_process_group()
