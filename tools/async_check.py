"""NEXT row f2 across ranks (torchrun; BOOTSTRAP as tools/multi_gpu_check.py): every rank hosts L_LOCAL
learners and one shard; gorila_async_run (collective) runs STEPS asynchronous learner steps per learner
while every rank's shard server applies the messages of all ranks' learners as they arrive.
Checks: every shard saw every message (fresh + stale = all ranks' sent), its version = its fresh count,
theta^+ gathered from the owners is identical on every rank, and it moved. Prints one JSON line per
rank with the counts (rank 0 last: "ASYNC CHECK OK")."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila, nccl_unique_id  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    ndev = torch.cuda.device_count()
    boot = os.environ.get("BOOTSTRAP", "nccl" if ndev >= world else "ipc")
    dev = local if boot == "nccl" else local % ndev
    torch.cuda.set_device(dev)
    if boot == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    else:
        dist.init_process_group("gloo")
        nid = None
    L, K = int(os.environ.get("L_LOCAL", "2")), int(os.environ.get("STEPS", "10"))
    nA, B, C = 6, 32, 2000
    g = Gorila(n_actions=nA, batch=B, replay_capacity=C, n_learners_local=L, learner_id_base=rank * L, rank=rank,
               world=world, nccl_unique_id=nid, theta0=synth.theta0(nA), math=os.environ.get("MATH", "bf16"),
               ps_mode="async", max_staleness=int(os.environ.get("MAX_DELAY", "2")), target_period=5,
               outlier_warmup=3)
    for j in range(L):
        gid = rank * L + j
        g.replay_insert(j, synth.frames(synth.SEED_DATA, gid, 0, C), *synth.meta(synth.SEED_DATA, gid, 0, C, nA))
    th0 = g.get_state()[0]
    st = g.async_run(list(range(L)), K, server_blocks=int(os.environ.get("SERVER_BLOCKS", "16")))
    th1, _, _, V = g.get_state()
    every = [None] * world
    dist.all_gather_object(every, {"rank": rank, **st, "theta1": th1})
    ok = True
    sent = sum(e["sent"] for e in every)
    for e in every:
        ok &= e["fresh"] + e["stale"] == sent and e["version_after"] == e["fresh"] and e["steps"] == K * L
        ok &= np.array_equal(e["theta1"], every[0]["theta1"])
    ok &= bool(np.all(np.isfinite(th1))) and not np.array_equal(th0, th1)
    flag = [None] * world
    dist.all_gather_object(flag, bool(ok))
    for e in every if rank == 0 else []:
        print(json.dumps({k: v for k, v in e.items() if k != "theta1"}), flush=True)
    g.close()
    dist.destroy_process_group()
    if rank == 0:
        print("ASYNC CHECK", "OK" if all(flag) else "FAILED", flush=True)
    sys.exit(0 if all(flag) else 1)


if __name__ == "__main__":
    main()
