"""Multi-rank parity check of the sharded parameter server (run under torchrun, one process per rank):

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/multi_gpu_check.py

BOOTSTRAP=nccl (default when there is one GPU per rank): rank r on cuda:r, the library's NCCL
communicator bootstraps the peer mappings. BOOTSTRAP=ipc (default with fewer GPUs than ranks): a
gloo process group, every rank on cuda:(r mod #GPUs) -- several ranks may share one GPU -- and the
CUDA IPC records of the workspaces are exchanged over gloo (gorila_peer_connect). Either way the
data path is the same peer-memory kernel (k_apply_p2p: gradient slices summed in rank order, the
optimizer on the owner's shard, the new replica chunk stored into every rank; Alg.1 P:116 /
P:129), plus k_replay_barrier / the peer gathers of the global replay (REPLAY=global, f4).

Rank r hosts L_LOCAL learners (global ids r*L_LOCAL + j) with their own synthetic replays. Every
round, rank 0 teacher-forces the oracle -- all N*L_LOCAL learners on one parameter server -- from
the GPU state (theta, the sharded m / v gathered from their owners, V, every learner's theta^- and
loss statistics) and checks, at BASELINE.json's tolerances (1e-5 fp32 / 1e-3 bf16 for Q and loss,
1e-5 / 5e-3 normalised L2 for gradients and updates): every learner's Q, Q-hat and loss on every
rank; decisions, accepted counts, versions and sync events exactly; each rank's gradient sum per
tensor (the oracle's backward teacher-forced to the GPU's ambiguous ReLU decisions, R30);
the update per tensor (R31 fp32-state floor; R33 in per-message mode). Every rank checks that the
theta^+ replicas are bitwise identical across ranks, and (REPLAY=global) its own draws bit-exact.
Prints "MULTI-GPU CHECK OK" on rank 0 and exits 0 iff every check on every rank passed.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import synth  # noqa: E402
from gpu_util import TOL, gpu_acts, per_tensor_rel_l2, rel_inf, rel_l2, teacher_forced_acts  # noqa: E402
from paper_1507_04296_b200 import Gorila, nccl_unique_id  # noqa: E402


def gather(obj, world):
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


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
    math = os.environ.get("MATH", "fp32")
    ps_mode = os.environ.get("PS_MODE", "aggregate")
    rounds = int(os.environ.get("ROUNDS", "4"))
    replay = os.environ.get("REPLAY", "local")
    Ll = int(os.environ.get("L_LOCAL", "1"))
    nA, B, C = 6, int(os.environ.get("BATCH", "16")), 1200  # BATCH >= 75: the large-batch (ring-gather) path
    G_ = world * Ll
    fill = (lambda j: [1500, 700, 1000, 400][j % 4]) if replay == "global" else (lambda j: C)
    tol = TOL[math]
    mode = "exact" if math == "fp32" else "bf16"
    theta0 = synth.theta0(nA)
    g = Gorila(n_actions=nA, batch=B, replay_capacity=C, n_learners_local=Ll, learner_id_base=rank * Ll, rank=rank,
               world=world, nccl_unique_id=nid, theta0=theta0, math=math, target_period=3, outlier_warmup=2,
               ps_mode=ps_mode, replay_mode=replay)
    g.capture_activations(True)
    for j in range(Ll):
        gid = rank * Ll + j
        f = synth.frames(synth.SEED_DATA, gid, 0, fill(gid))
        a, r, d = synth.meta(synth.SEED_DATA, gid, 0, fill(gid), nA)
        g.replay_insert(j, f, a, r, d)
    rings = None
    if replay == "global":  # every rank holds the oracle's copy of all rings to check its own draws
        rings = []
        for j in range(G_):
            rg = O.Ring(C)
            rg.insert(synth.frames(synth.SEED_DATA, j, 0, fill(j)), *synth.meta(synth.SEED_DATA, j, 0, fill(j), nA))
            rings.append(rg)
    orc = None
    if rank == 0:
        orc = O.GorilaOracle(O.Config(n_actions=nA, batch=B, capacity=C, learners=tuple(range(G_)), mode=mode,
                                      target_period=3, outlier_warmup=2, ps_mode=ps_mode, replay_mode=replay,
                                      n_shards=world), theta0)
        for j in range(G_):
            orc.insert(j, synth.frames(synth.SEED_DATA, j, 0, fill(j)), *synth.meta(synth.SEED_DATA, j, 0, fill(j), nA))
    fails = []
    ids = list(range(Ll))
    for k in range(rounds):
        if rings is not None:  # f4: this rank's draws, bit-exact (replay_sample is collective here)
            for j in ids:
                gs = g.replay_sample(j, k)
                shard, tau = O.sample_indices_global([rg.n for rg in rings], C, B, 1507, rank * Ll + j, k)
                s_, s2_, a_, r_, d_ = O.gather_global(rings, shard, tau)
                same = (np.array_equal(g.replay_sample_shards(), shard) and np.array_equal(gs["tau"], tau) and
                        np.array_equal(gs["s"], s_) and np.array_equal(gs["s2"], s2_) and
                        np.array_equal(gs["a"], a_) and np.array_equal(gs["r"], r_) and np.array_equal(gs["d"], d_))
                if not same:
                    fails.append(f"rank {rank} learner {j} round {k}: global draw differs")
        # the state every rank starts the round from (teacher forcing of the oracle)
        th0, m0, v0, V0 = g.get_state()
        lstate = {rank * Ll + j: g.get_learner_state(j) for j in ids}
        # one round (learner_step + ps_apply_shard + sync_target; records read after it, when the
        # per-message PS decisions are final); G, Q and the captured activations are intact after it
        info, ri, synced = g.round(np.array(ids, np.int32), k, want_info=True)
        qs = {rank * Ll + j: g.get_q(j) for j in ids}
        acts = {rank * Ll + j: gpu_acts(g, j) for j in ids if not info[j]["not_ready"]}
        Gr = g.get_grad()
        th1, _, _, V1 = g.get_state()
        allth = gather(th1, world)
        if not all(np.array_equal(allth[0], x) for x in allth):
            fails.append(f"rank {rank} round {k}: theta+ replicas differ across ranks")
        mine = {"m": m0, "v": v0, "lstate": lstate, "info": {rank * Ll + j: info[j] for j in ids}, "q": qs,
                "acts": acts, "G": Gr, "ri": ri, "synced": {rank * Ll + j: bool(synced[j]) for j in ids}}
        every = gather(mine, world)
        if rank == 0:
            # teacher forcing: theta, V from rank 0 (identical everywhere), m / v from their owners (each
            # rank returns its own slice, zeros elsewhere), every learner's theta^- and statistics
            orc.theta = th0.astype(np.float64)
            orc.m = sum(e["m"].astype(np.float64) for e in every)
            orc.v = sum(e["v"].astype(np.float64) for e in every)
            orc.V = int(V0)
            orc.history = {}
            acts_all, infos, qall, synced_all = {}, {}, {}, {}
            for e in every:
                acts_all.update(e["acts"])
                infos.update(e["info"])
                qall.update(e["q"])
                synced_all.update(e["synced"])
                for gid, (tm, st) in e["lstate"].items():
                    L_ = orc.learners[gid]
                    L_.theta_minus = tm.astype(np.float64)
                    L_.stats = O.LossStats(mu=st["mu"], var=st["var"], count=st["count"])
                    L_.last_sync = st["last_sync"]
            forced = []
            res = orc.round(k, acts_hook=lambda gid, a_, z_: teacher_forced_acts(acts_all[gid], a_, z_, math, forced))
            for gid in range(G_):
                gi, oi = infos[gid], res["learners"][gid]
                for key in ("accepted", "stale", "not_ready"):
                    if bool(gi[key]) != bool(oi[key]):
                        fails.append(f"round {k} learner {gid}: {key} {gi[key]} vs oracle {oi[key]}")
                if oi["not_ready"]:
                    continue
                thr = oi["threshold"]
                if (oi["stats_count_before"] < 1 or abs(oi["abs_loss"] - thr) > 1e-2 * abs(thr)) and \
                        bool(gi["rejected_outlier"]) != bool(oi["rejected_outlier"]):
                    fails.append(f"round {k} learner {gid}: outlier decision differs")
                q, qh = qall[gid]
                eq, eqh = rel_inf(q, oi["Q"]), rel_inf(qh, oi["Qhat"])
                el = abs(gi["loss"] - oi["loss"]) / max(abs(oi["loss"]), 1e-12)
                if eq > tol["q"] or eqh > tol["q"] or el > tol["loss"]:
                    fails.append(f"round {k} learner {gid}: Q {eq:.2e} Qhat {eqh:.2e} loss {el:.2e}")
            for q_rank, e in enumerate(every):  # each rank's gradient sum, per tensor
                ref = np.zeros(len(th0))
                for gid in range(q_rank * Ll, (q_rank + 1) * Ll):
                    oi = res["learners"][gid]
                    # per-message mode judges staleness at the PS: every sent message's gradient is there
                    if oi["accepted"] or (ps_mode == "per_message" and "G" in oi):
                        ref += oi["G"]
                if not np.any(ref):
                    if np.any(e["G"]):
                        fails.append(f"round {k} rank {q_rank}: nonzero G without an accepted learner")
                    continue
                errs = per_tensor_rel_l2(e["G"], ref, nA)
                bad = {n_: v_ for n_, v_ in errs.items() if v_ > tol["g"]}
                if bad and os.environ.get("DEBUG_G"):
                    for gid in range(q_rank * Ll, (q_rank + 1) * Ll):
                        oi = res["learners"][gid]
                        print(f"  dbg round {k} gid {gid}: gpu {infos[gid]} oracle acc {oi['accepted']} "
                              f"rej {oi['rejected_outlier']} stale {oi['stale']} hasG {'G' in oi}", flush=True)
                        if "G" in oi:
                            print("   vs this learner alone:", {n_: round(v_, 4) for n_, v_ in
                                                                per_tensor_rel_l2(e["G"], oi["G"], nA).items()}, flush=True)
                if rel_l2(e["G"], ref) > tol["g"] or bad:
                    fails.append(f"round {k} rank {q_rank}: G {rel_l2(e['G'], ref):.2e} per tensor {bad}")
            ri0 = every[0]["ri"]
            if ri0["n_accepted"] != res["n_accepted"] or V1 != res["version_after"]:
                fails.append(f"round {k}: n_acc {ri0['n_accepted']} V {V1} vs oracle {res['n_accepted']} "
                             f"{res['version_after']}")
            if any(synced_all[gid] != bool(res["synced"][gid]) for gid in range(G_)):
                fails.append(f"round {k}: sync events differ")
            # the update per tensor: fp32-state floor (R31), once per optimizer step (R33)
            n_msg = max(1, res["n_accepted"]) if ps_mode == "per_message" else 1
            n_round = n_msg + 1 if ps_mode == "per_message" else 1
            tol_d = max(tol["dtheta"], n_msg * tol["g"]) if ps_mode == "per_message" else tol["dtheta"]
            d_gpu = th1.astype(np.float64) - th0
            th1_ref = orc.theta.astype(np.float32)
            d_ref = th1_ref.astype(np.float64) - th0
            ulp = np.spacing(np.abs(th1_ref)).astype(np.float64)
            off, worst = 0, 0.0
            for name, shp in O.param_shapes(nA):
                n = int(np.prod(shp))
                sl = slice(off, off + n)
                off += n
                if not np.any(d_ref[sl]):
                    if np.any(d_gpu[sl]):
                        fails.append(f"round {k}: {name} moved without an update")
                    continue
                e_ = rel_l2(d_gpu[sl], d_ref[sl])
                floor = n_round * np.linalg.norm(ulp[sl]) / np.linalg.norm(d_ref[sl])
                worst = max(worst, e_ / (tol_d + floor))
                if e_ > tol_d + floor:
                    fails.append(f"round {k}: dtheta {name} {e_:.2e} > {tol_d + floor:.2e}")
            print(f"round {k}: V {V1} acc {res['n_accepted']} synced {sum(synced_all.values())} "
                  f"worst dtheta/bound {worst:.2f} forced {forced}", flush=True)
    allf = gather(fails, world)
    g.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        flat = [x for f in allf for x in f]
        for x in flat[:40]:
            print("FAIL", x, flush=True)
        print(f"world {world} bootstrap {boot} devices {ndev} math {math} ps {ps_mode} replay {replay} "
              f"learners/rank {Ll}", flush=True)
        print("MULTI-GPU CHECK", "OK" if not flat else "FAILED", flush=True)
    sys.exit(0 if not any(allf) else 1)


if __name__ == "__main__":
    main()
