"""Multi-GPU parity check (run under torchrun, one rank per GPU):

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/multi_gpu_check.py

Every rank hosts one learner (global id = rank) with its own synthetic replay and a 1/N
parameter-server shard (NCCL reduce-scatter / all-gather inside ps_apply_shard). Rank 0
runs the CPU oracle with all N learners on one parameter server and checks, each round:
decisions and versions exactly, Q of its own learner, and the parameter update (normalised
L2 of the update, fp32 check mode: 1e-5 + the fp32 state floor). All ranks check that their
theta+ replicas are bitwise identical after the all-gather. Exits non-zero on failure.
REPLAY=global (NEXT row f4): every learner draws from the union of all ranks' rings (unequal
fills, one wrapped), gathered over NVLink; each rank also checks its own draw (shard, tau,
frames, a / r / d) bit-exact against the oracle's global draw.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila, nccl_unique_id  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    math = os.environ.get("MATH", "fp32")
    ps_mode = os.environ.get("PS_MODE", "aggregate")  # "per_message": NEXT row f1 over the peer-memory exchange
    rounds = int(os.environ.get("ROUNDS", "4"))
    replay = os.environ.get("REPLAY", "local")
    fill = (lambda j: [1500, 700, 1000, 400][j % 4]) if replay == "global" else (lambda j: C)
    nA, B, C = 6, 16, 1200
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    theta0 = synth.theta0(nA)
    g = Gorila(n_actions=nA, batch=B, replay_capacity=C, n_learners_local=1, learner_id_base=rank, rank=rank,
               world=world, nccl_unique_id=obj[0], theta0=theta0, math=math, target_period=3, outlier_warmup=2,
               ps_mode=ps_mode, replay_mode=replay)
    f = synth.frames(synth.SEED_DATA, rank, 0, fill(rank))
    a, r, d = synth.meta(synth.SEED_DATA, rank, 0, fill(rank), nA)
    g.replay_insert(0, f, a, r, d)
    rings = None
    if replay == "global":  # every rank holds the oracle's copy of all rings to check its own draws
        rings = []
        for j in range(world):
            rg = O.Ring(C)
            rg.insert(synth.frames(synth.SEED_DATA, j, 0, fill(j)), *synth.meta(synth.SEED_DATA, j, 0, fill(j), nA))
            rings.append(rg)
    orc = None
    if rank == 0:
        orc = O.GorilaOracle(O.Config(n_actions=nA, batch=B, capacity=C, learners=tuple(range(world)),
                                      mode="exact" if math == "fp32" else "bf16", target_period=3,
                                      outlier_warmup=2, ps_mode=ps_mode, replay_mode=replay), theta0)
        for j in range(world):
            fj = synth.frames(synth.SEED_DATA, j, 0, fill(j))
            aj, rj, dj = synth.meta(synth.SEED_DATA, j, 0, fill(j), nA)
            orc.insert(j, fj, aj, rj, dj)
    ok = True
    tol = 1e-5 if math == "fp32" else 5e-3
    for k in range(rounds):
        if rings is not None:  # f4: this rank's draw, bit-exact (replay_sample is collective here)
            gs = g.replay_sample(0, k)
            shard, tau = O.sample_indices_global([rg.n for rg in rings], C, B, 1507, rank, k)
            s_, s2_, a_, r_, d_ = O.gather_global(rings, shard, tau)
            same = (np.array_equal(g.replay_sample_shards(), shard) and np.array_equal(gs["tau"], tau) and
                    np.array_equal(gs["s"], s_) and np.array_equal(gs["s2"], s2_) and np.array_equal(gs["a"], a_)
                    and np.array_equal(gs["r"], r_) and np.array_equal(gs["d"], d_))
            print(f"[rank {rank}] round {k}: global draw shards {np.bincount(shard, minlength=world).tolist()} "
                  f"{'bit-exact' if same else 'MISMATCH'}", flush=True)
            ok = ok and same
        th0 = g.get_state()[0]
        info = g.learner_step([0], k)[0]
        q = g.get_q(0)[0]
        ri = g.ps_apply_shard(k)
        synced = bool(g.sync_target([0])[0])
        th1, _, _, V = g.get_state()
        # replicas identical on every rank after the all-gather
        h = torch.from_numpy(th1).cuda()
        hs = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        if not all(torch.equal(hs[0], x) for x in hs):
            print(f"[rank {rank}] round {k}: theta+ replicas differ across ranks", flush=True)
            ok = False
        infos = [None] * world
        dist.all_gather_object(infos, {"accepted": info["accepted"], "stale": info["stale"],
                                       "rejected": info["rejected_outlier"], "loss": info["loss"]})
        if rank == 0:
            res = orc.round(k)
            for j in range(world):
                oi = res["learners"][j]
                if bool(infos[j]["accepted"]) != bool(oi["accepted"]) or bool(infos[j]["stale"]) != bool(oi["stale"]):
                    print(f"round {k} learner {j}: decision mismatch {infos[j]} vs oracle", flush=True)
                    ok = False
                if abs(infos[j]["loss"] - oi["loss"]) > (1e-4 if math == "fp32" else 2e-3) * abs(oi["loss"]):
                    print(f"round {k} learner {j}: loss {infos[j]['loss']} vs {oi['loss']}", flush=True)
                    ok = False
            eq = np.max(np.abs(q - res["learners"][0]["Q"])) / np.max(np.abs(res["learners"][0]["Q"]))
            if ri["n_accepted"] != res["n_accepted"] or V != res["version_after"] or synced != res["synced"][0]:
                print(f"round {k}: counts {ri} V {V} synced {synced} vs oracle {res['n_accepted']} "
                      f"{res['version_after']} {res['synced'][0]}", flush=True)
                ok = False
            d_gpu = th1.astype(np.float64) - th0
            d_ref = orc.theta.astype(np.float32).astype(np.float64) - th0
            n_msg = max(1, res["n_accepted"]) if ps_mode == "per_message" else 1
            n_round = n_msg + 1 if ps_mode == "per_message" else 1  # R33
            floor = n_round * np.linalg.norm(np.spacing(np.abs(orc.theta.astype(np.float32)))) / np.linalg.norm(d_ref)
            e = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
            print(f"round {k}: Q err {eq:.2e}  dtheta err {e:.2e} (bound {tol + floor:.2e})  V {V}  "
                  f"acc {ri['n_accepted']}  synced {synced}", flush=True)
            tol_d = max(tol, n_msg * (1e-5 if math == "fp32" else 5e-3)) if ps_mode == "per_message" else tol
            if eq > (1e-4 if math == "fp32" else 1e-3) or e > tol_d + floor:
                ok = False
            # teacher-force: continue from the GPU state (m, v are sharded: keep the oracle's)
            orc.theta = th1.astype(np.float64)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    g.close()
    dist.destroy_process_group()
    if rank == 0:
        print("MULTI-GPU CHECK", "OK" if flag.item() == 1 else "FAILED", flush=True)
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
