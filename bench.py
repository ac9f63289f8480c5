#!/usr/bin/env python
"""Benchmark: DQN learner updates/sec (batch 32) of the B200-native Gorila learner update.

Workload (BASELINE.json configs[1]): one learner per GPU, |A| = 18, batch 32, a 1M-frame
device replay (synthetic Atari-shaped frames, synth/), RMSProp parameter server sharded over
the ranks, target sync every 100 PS updates. A step = learner_step + ps_apply_shard +
sync_target (the whole hot path: sample -> 2 forwards -> TD -> backward -> [reduce-scatter]
-> RMSProp -> [all-gather] -> replica -> target sync).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun (N > 1) every rank runs one learner; rank 0 prints ONE JSON line.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DQN learner updates/sec (batch 32)"
UNIT = "updates/s"

# algorithmic work per learner update, per sample
MAC = {"conv1": 3_276_800, "conv2": 2_654_208, "conv3": 1_806_336, "fc4": 1_605_632}


def fc5_mac(nA):
    return 512 * nA


def phase_work(phase, B, nA, P, esz, n_msg=1, tower=False):
    """(bound, algorithmic amount per launch-group, unit) of a profiled phase. n_msg: gradient
    buffers the apply reads (per-message mode reads one per local learner). tower: the small-batch
    conv tower runs conv1..conv3 of both nets inside the conv1_fwd phase."""
    fl = lambda mac: 2.0 * mac * B  # noqa: E731
    if tower and phase in ("conv2_fwd", "conv3_fwd"):
        return None
    if tower and phase == "conv1_fwd":
        return ("tensor", 2 * fl(MAC["conv1"] + MAC["conv2"] + MAC["conv3"]))
    table = {
        "conv1_fwd": ("tensor", 2 * fl(MAC["conv1"])), "conv2_fwd": ("tensor", 2 * fl(MAC["conv2"])),
        "conv3_fwd": ("tensor", 2 * fl(MAC["conv3"])), "fc4_fwd": ("tensor", 2 * fl(MAC["fc4"])),
        "fc4_dgrad": ("tensor", fl(MAC["fc4"])), "fc4_wgrad": ("tensor", fl(MAC["fc4"])),
        "conv3_dgrad": ("tensor", fl(MAC["conv3"])), "conv3_wgrad": ("tensor", fl(MAC["conv3"])),
        "conv2_dgrad": ("tensor", fl(MAC["conv2"])), "conv2_wgrad": ("tensor", fl(MAC["conv2"])),
        "conv1_wgrad": ("tensor", fl(MAC["conv1"])),
        # sampler: reads 5 frames + meta per sample, writes s and s' (NHWC, esz bytes/element)
        "sample": ("hbm", B * (5 * 7056 + 6 + 2 * 4 * 7056 * esz)),
        # centered RMSProp: read theta, m, v, g (16 B) + write theta, m, v (12 B) per parameter, plus the
        # fused emission of the next replica (esz bytes per parameter)
        "apply": ("hbm", (28.0 + esz + 4.0 * (n_msg - 1)) * P),
        # replica pack (world > 1, after the all-gather): read fp32 theta, write the replica
        "pack": ("hbm", (4.0 + esz) * P),
    }
    return table.get(phase)


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return {"hbm": float(pk["hbm_gbs"]), "tensor": float(pk["bf16_tflops_sustained"]),
                "tensor_burst": float(pk["bf16_tflops"]), "src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm": 6650.0, "tensor": 1400.0, "tensor_burst": 1590.0, "src": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML (nvidia_ml_py) in a
    background thread every 20 ms, nvidia-smi's loop mode as the fallback (B200_PROFILING.md clocks
    line). summary() reports the samples taken while the device was busy with the bench."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []  # (sm_mhz, max_mhz, reasons)
        self.failures = 0  # NVML queries that raised
        self.src = None
        self.proc = None
        self.stop = None
        self.f = None

    def _nvml_loop(self, h, nv):
        import time as _t
        try:
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception:
            mx = float("nan")
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            except Exception:
                self.failures += 1
                _t.sleep(0.02)
                continue
            reasons = set()
            try:  # a failed reasons query still records the clock (and is counted)
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                reasons = {k for k, bit in self.BITS.items() if r & bit}
            except Exception:
                self.failures += 1
            self.rows.append((float(sm), mx, reasons))
            _t.sleep(0.02)

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.idx]) if vis and vis.split(",")[0].isdigit() else self.idx
            h = nv.nvmlDeviceGetHandleByIndex(phys)
            self.stop = threading.Event()
            self.th = threading.Thread(target=self._nvml_loop, args=(h, nv), daemon=True)
            self.th.start()
            self.src = "nvml"
            return self
        except Exception:
            pass
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
            self.src = "nvidia-smi"
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.stop is not None:
            self.stop.set()
            self.th.join()
            if not self.rows:  # every NVML query failed: one nvidia-smi sample right after the loop
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=20).stdout
                    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                    for r in [r.split(",") for r in out.strip().splitlines() if r.strip()]:
                        self.rows.append((float(r[1]), float(r[2]),
                                          {names[i] for i in range(4) if len(r) > 5 + i and r[5 + i].strip() == "Active"}))
                    self.src = "nvidia-smi (after the loop: NVML failed)"
                except Exception:
                    pass
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.flush()
            self.f.seek(0)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for r in [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]:
                try:
                    self.rows.append((float(r[1]), float(r[2]),
                                      {names[i] for i in range(4) if len(r) > 5 + i and r[5 + i].strip() == "Active"}))
                except (ValueError, IndexError):
                    pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0,
                    "src": self.src, "query_failures": self.failures}
        sm = [r[0] for r in self.rows]
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
               "reasons": sorted(set().union(*[r[2] for r in self.rows])), "samples": len(self.rows),
               "src": self.src}
        if self.failures:
            out["query_failures"] = self.failures
        return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def fill_replay(g, learner, capacity, n_actions, seed, learner_gid, chunk=131072, p_poison=0.0):
    import torch
    import synth
    fr = torch.empty((chunk, 84, 84), dtype=torch.uint8, device="cuda")
    a = torch.empty(chunk, dtype=torch.uint8, device="cuda")
    r = torch.empty(chunk, dtype=torch.float32, device="cuda")
    d = torch.empty(chunk, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    t = 0
    while t < capacity:
        n = min(chunk, capacity - t)
        synth.fill_frames_dev(seed, learner_gid, t, n, fr.data_ptr(), st)
        synth.fill_meta_dev(seed, learner_gid, t, n, n_actions, p_poison, a.data_ptr(), r.data_ptr(), d.data_ptr(), st)
        g.replay_insert(learner, fr[:n], a[:n], r[:n], d[:n])
        t += n
    torch.cuda.synchronize()


def cpu_baseline(args, budget_s):
    """The oracle (as it stands) on the host cores: a bounded sample of the same workload."""
    import oracle as O
    import synth
    nA, B = args.n_actions, args.batch
    cap = 20_000
    cfg = O.Config(n_actions=nA, batch=B, capacity=cap, mode="exact", target_period=args.target_period)
    orc = O.GorilaOracle(cfg, synth.theta0(nA))
    f = synth.frames(synth.SEED_DATA, 0, 0, cap)
    a, r, d = synth.meta(synth.SEED_DATA, 0, 0, cap, nA)
    orc.insert(0, f, a, r, d)
    orc.round(0)  # warm-up (page-in, OpenMP pool)
    t0 = time.perf_counter()
    k = 1
    while True:
        orc.round(k)
        k += 1
        el = time.perf_counter() - t0
        if el >= budget_s or k > 200:
            break
    n = k - 1
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": n / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n} oracle learner updates (nA={nA}, B={B}, fp64, {cores} OpenMP threads) on a "
                      f"{cap}-frame replay (per-update work does not depend on replay size), {el:.1f} s"}


C1_SCRIPT = r"""
import os, sys, time
sys.path.insert(0, {root!r})
import oracle as O, synth
cfg = O.Config(n_actions=4, batch=32, capacity=10_000, mode="exact", target_period=100)
orc = O.GorilaOracle(cfg, synth.theta0(4))
f = synth.frames(synth.SEED_DATA, 0, 0, 10_000)
a, r, d = synth.meta(synth.SEED_DATA, 0, 0, 10_000, 4)
orc.insert(0, f, a, r, d)
t0 = time.perf_counter()
for k in range(10):
    orc.round(k)
print("C1_SECONDS", time.perf_counter() - t0)
"""


def c1_timing(g_factory):
    """BASELINE configs[0] (C1: nA=4, B=32, 10k transitions, 10 RMSProp steps) in seconds: the oracle as it
    stands at 1 OpenMP thread and at nproc threads (separate processes so the OpenMP
    runtime takes each thread count), and the GPU path's device time for the same 10 rounds."""
    out = {"nproc": os.cpu_count(), "cpu_model": None}
    try:
        with open("/proc/cpuinfo") as f:
            out["cpu_model"] = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), None)
    except OSError:
        pass
    for key, threads in (("oracle_s_1thread", 1), ("oracle_s_nproc", os.cpu_count() or 1)):
        env = dict(os.environ, OMP_NUM_THREADS=str(threads))
        r = subprocess.run([sys.executable, "-c", C1_SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                           timeout=600)
        vals = [l.split()[1] for l in r.stdout.splitlines() if l.startswith("C1_SECONDS")]
        out[key] = float(vals[0]) if vals else None
    out["gpu_s"] = g_factory()
    out["note"] = "10 learner updates of configs[0]; oracle wall clock (steady perf_counter) per process; GPU: " \
                  "device time of 10 graph rounds after 10 warm-up rounds (CUDA events)"
    return out


def gpu_c1_seconds():
    import torch
    import synth
    from paper_1507_04296_b200 import Gorila
    st = torch.cuda.current_stream()
    g = Gorila(n_actions=4, batch=32, replay_capacity=10_000, theta0=synth.theta0(4), stream=st, math="bf16")
    f = synth.frames(synth.SEED_DATA, 0, 0, 10_000)
    a, r, d = synth.meta(synth.SEED_DATA, 0, 0, 10_000, 4)
    g.replay_insert(0, f, a, r, d)
    ids = np.zeros(1, np.int32)
    for k in range(10):
        g.round(ids, k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.synchronize()
    e0.record(st)
    for k in range(10, 20):
        g.round(ids, k)
    e1.record(st)
    st.synchronize()
    g.close()
    return e0.elapsed_time(e1) / 1000.0


def run_reference(args, json_out):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    import synth
    nA, B = args.n_actions, args.batch
    cap = 20_000
    cfg = O.Config(n_actions=nA, batch=B, capacity=cap, mode="exact", target_period=args.target_period)
    orc = O.GorilaOracle(cfg, synth.theta0(nA))
    f = synth.frames(synth.SEED_DATA, 0, 0, cap)
    a, r, d = synth.meta(synth.SEED_DATA, 0, 0, cap, nA)
    orc.insert(0, f, a, r, d)
    t1 = time.perf_counter()
    orc.round(0)
    one = time.perf_counter() - t1
    warm = min(args.warmup, 3)
    for k in range(1, warm):
        orc.round(k)
    budget = 150.0
    steps = int(max(3, min(args.steps, budget // max(one, 1e-3))))
    t0 = time.perf_counter()
    for k in range(steps):
        orc.round(warm + k)
    el = time.perf_counter() - t0
    val = steps / el
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    sample = (f"{steps} oracle learner updates (of --steps {args.steps}; bounded to ~{int(budget)} s) nA={nA} "
              f"B={B} fp64 on a {cap}-frame replay")
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
                      "steps": steps, "warmup": warm, "ms_per_step": 1000 * el / steps, "higher_is_better": True,
                      "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": config_dict(args, world),
                      "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
                      "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          file=json_out, flush=True)


def config_dict(args, world):
    if args.learners == 1 and args.batch == 32 and args.capacity == 1_000_000 and args.target_period == 100:
        wl = "configs[1]: 1 learner/GPU, |A|=18, batch 32, 1M-frame device replay, target sync every 100"
    elif args.learners > 1:
        wl = (f"configs[4]-shaped: {args.learners} logical learners/GPU, batch {args.batch}, {args.capacity}-frame "
              f"replay each, target sync every {args.target_period}, scheduled staleness {args.staleness}, "
              f"max delay {args.max_staleness}, poison {args.poison}")
    else:
        wl = f"configs[3] sweep point: 1 learner/GPU, batch {args.batch}, {args.capacity}-frame replay"
    if args.replay == "global":
        wl += "; global replay (NEXT row f4): every batch drawn from the union of all learners' rings on all GPUs"
    return {"workload": wl, "replay": args.replay,
            "n_actions": args.n_actions, "batch_per_learner": args.batch, "learners_per_gpu": args.learners,
            "global_batch": args.batch * world * args.learners,
            "replay_frames_per_learner": args.capacity, "target_period": args.target_period,
            "ps_mode": args.ps_mode, "optimizer": args.optimizer,
            "ps_shards": world, "parallelism": f"dp{world} learners + {world}-way sharded PS "
                                               f"({'NVLink peer-memory exchange' if world > 1 else 'local'})",
            "math": args.math, "l2": "inputs larger than L2: 7.06 GB replay per GPU (126 MB L2); the 27 MB "
                                     "parameter/optimizer state stays L2-resident across steps as in training"}


def run_async(args, g, ids, world, rank, local_rank, json_out):
    """NEXT row f2: learner steps/s of gorila_async_run (learners and shard servers decoupled), device-timed
    around the call on the library stream, max over ranks; the shards' accept / stale counts and the
    learners' outlier rejections of the timed run."""
    import torch
    L = len(ids)
    stream = g.stream
    g.async_run(ids, args.warmup, round0=0, server_blocks=args.server_blocks)  # warm-up (also loads kernels)
    barrier(world)
    clk = ClockSampler(local_rank).__enter__()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream.synchronize()
    barrier(world)
    e0.record(stream)
    st = g.async_run(ids, args.steps, round0=args.warmup, server_blocks=args.server_blocks)
    e1.record(stream)
    stream.synchronize()
    clk.__exit__(None, None, None)
    ms = max_over_ranks(e0.elapsed_time(e1), world) if args.bootstrap == "nccl" else e0.elapsed_time(e1)
    if world > 1 and args.bootstrap == "ipc":
        import torch.distributed as dist
        allms = [None] * world
        dist.all_gather_object(allms, ms)
        ms = max(allms)
    stats = [st]
    if world > 1:
        import torch.distributed as dist
        stats = [None] * world
        dist.all_gather_object(stats, st)
    value = world * L * args.steps / (ms / 1000.0)
    if rank == 0:
        cfg = config_dict(args, world)
        cfg["workload"] += "; NEXT row f2: asynchronous PS (gorila_async_run), learner steps counted"
        cfg["bootstrap"] = args.bootstrap
        cfg["server_blocks"] = args.server_blocks
        out = {"metric": METRIC + " [asynchronous PS, f2]", "value": value, "unit": UNIT, "n_gpus": world,
               "gpus_physical": torch.cuda.device_count() if args.bootstrap == "ipc" else world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if args.math == "bf16" else "f32",
               "data": "synthetic", "config": cfg, "clocks": clk.summary(),
               "async": {"per_shard": stats,
                         "sent": sum(s["sent"] for s in stats), "rejected_outlier": sum(s["rejected"] for s in stats),
                         "fresh_per_shard": [s["fresh"] for s in stats], "stale_per_shard": [s["stale"] for s in stats],
                         "stale_fraction": [s["stale"] / max(1, s["fresh"] + s["stale"]) for s in stats],
                         "note": "one message per shard per non-rejected learner step; each shard judges staleness "
                                 "against its own live version (V_arrival - base > max_delay is discarded)"}}
        print(json.dumps(out), file=json_out, flush=True)
    g.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    # the contract's stdout is ONE JSON line: everything else (NCCL banners, warnings) goes to stderr
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--math", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--n-actions", type=int, default=18)
    ap.add_argument("--capacity", type=int, default=1_000_000)
    ap.add_argument("--target-period", type=int, default=100)
    ap.add_argument("--learners", type=int, default=1, help="logical learners per GPU (configs[4]: 12-25)")
    ap.add_argument("--staleness", type=int, default=0, help="scheduled staleness of every learner (rounds)")
    ap.add_argument("--max-staleness", type=int, default=-1, help="discard threshold in versions (-1: off)")
    ap.add_argument("--poison", type=float, default=0.0, help="probability of a 1e6 poison reward")
    ap.add_argument("--ps-mode", default="aggregate", choices=["aggregate", "per_message", "async"],
                    help="per_message: NEXT row f1 (one optimizer step per accepted learner gradient); "
                         "async: NEXT row f2 (learners and shard servers decoupled, gorila_async_run)")
    ap.add_argument("--bootstrap", default="nccl", choices=["nccl", "ipc"],
                    help="ipc: gloo process group + caller-exchanged peer mappings (several ranks may share "
                         "one GPU: rank r on cuda:(r mod #GPUs))")
    ap.add_argument("--server-blocks", type=int, default=32, help="async: blocks of each shard's server kernel")
    ap.add_argument("--optimizer", default="rmsprop", choices=["rmsprop", "adagrad"])
    ap.add_argument("--replay", default="local", choices=["local", "global"],
                    help="global: NEXT row f4 (uniform over all learners' rings, NVLink gathers)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1000)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        return run_reference(args, json_out)

    import torch
    world, rank, local_rank = dist_env()
    if args.bootstrap == "ipc":
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        if args.bootstrap == "ipc":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import synth
    from paper_1507_04296_b200 import Gorila, nccl_unique_id
    synth.build()
    uid = None
    if world > 1 and args.bootstrap == "nccl":
        import torch.distributed as dist
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    L = args.learners
    g = Gorila(n_actions=args.n_actions, batch=args.batch, replay_capacity=args.capacity, n_learners_local=L,
               learner_id_base=rank * L, rank=rank, world=world, nccl_unique_id=uid, stream=stream,
               theta0=synth.theta0(args.n_actions), math=args.math, target_period=args.target_period,
               history=max(2, args.staleness + 1), max_staleness=args.max_staleness, ps_mode=args.ps_mode, replay_mode=args.replay,
               optimizer=args.optimizer)
    for j in range(L):
        fill_replay(g, j, args.capacity, args.n_actions, synth.SEED_DATA, rank * L + j, p_poison=args.poison)
    ids = np.arange(L, dtype=np.int32)
    stal = np.full(L, args.staleness, np.int32) if args.staleness else None
    if args.ps_mode == "async":
        return run_async(args, g, ids, world, rank, local_rank, json_out)

    def step(k):
        g.round(ids, k, stal)  # learner_step + ps_apply_shard + sync_target, replayed as one CUDA graph

    def step_eager(k):
        g.learner_step_async(ids, k)
        g.ps_apply_shard(k, want_info=False)
        g.sync_target(ids, want_info=False)

    # clocks: sampled from the warm-up through the end-to-end loop (the timed region alone can be
    # shorter than one sampling period)
    clk = ClockSampler(local_rank).__enter__()
    k = 0
    for _ in range(args.warmup):
        step(k)
        k += 1
    # the timed region must contain target syncs (every target_period versions, one per accepted round
    # here): with fewer timed steps than the period, run untimed rounds up to half a period before a sync
    if args.steps < args.target_period and args.learners == 1:
        for _ in range(max(0, args.target_period - k - args.steps // 2)):
            step(k)
            k += 1
    stream.synchronize()
    barrier(world)
    sync0 = g.get_learner_state(0)[1]["last_sync"]
    V0 = g.get_state()[3]

    # ---------------- timed region (device time, CUDA events on the launching stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = g.kernel_launches()
    stream.synchronize()
    barrier(world)
    ev0.record(stream)
    for _ in range(args.steps):
        step(k)
        k += 1
    ev1.record(stream)
    stream.synchronize()
    barrier(world)
    launches = g.kernel_launches() - launches0
    sync1 = g.get_learner_state(0)[1]["last_sync"]
    V1 = g.get_state()[3]
    ms_local = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms_local, world)
    value = world * L * args.steps / (ms / 1000.0)

    # ---------------- end to end through the public API with host buffers
    f1 = torch.empty((1, 84, 84), dtype=torch.uint8).pin_memory()
    a1 = torch.zeros(1, dtype=torch.uint8).pin_memory()
    r1 = torch.zeros(1, dtype=torch.float32).pin_memory()
    d1 = torch.zeros(1, dtype=torch.uint8).pin_memory()
    n_e2e = args.warmup + args.e2e_steps
    hf = synth.frames(synth.SEED_DATA, rank, args.capacity, n_e2e)
    ha, hr, hd = synth.meta(synth.SEED_DATA, rank, args.capacity, n_e2e, args.n_actions)

    def e2e_step(i, k, pending):
        f1.numpy()[0] = hf[i]
        a1.numpy()[0], r1.numpy()[0], d1.numpy()[0] = ha[i], hr[i], hd[i]
        g.replay_insert(0, f1, a1, r1, d1)           # this step's new experience, pinned host -> device
        h = g.round_async(ids, k, stal)               # the round; its result (loss, decisions) -> pinned ring
        if pending is not None:
            g.round_result(pending)                   # the previous round's result, read while this one runs
        return h

    pending = None
    for i in range(args.warmup):                      # untimed warm-up of the same loop
        pending = e2e_step(i, k, pending)
        k += 1
    g.round_result(pending)
    barrier(world)
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pending = None
    for i in range(args.warmup, n_e2e):
        pending = e2e_step(i, k, pending)
        k += 1
    info = g.round_result(pending)
    e1.record(stream)
    stream.synchronize()
    clk.__exit__(None, None, None)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    e2e_value = world * L * args.e2e_steps / (e2e_ms / 1000.0)
    _ = info

    # ---------------- per-phase device timing (roofline of the dominant kernel)
    g.profile_enable(True)
    prof_steps = min(args.steps, 300)
    stream.synchronize()
    for _ in range(prof_steps):
        step(k)  # graph replay with event-record nodes between phases
        k += 1
    phases, n_prof = g.profile_read()
    g.profile_enable(False)
    # per-phase marginal device time, kernels re-launched back to back (warm L2, PDL as in the round)
    iso = {}
    for ph in phases:
        # not kernels of the round: td / misc are markers, the replica pack is fused into the apply
        # (1 GPU) or the peer-memory exchange (N > 1); RS / AG are the NCCL fallback's
        if ph in ("td", "step_misc", "reduce_scatter", "all_gather", "pack"):
            continue
        iso[ph] = g.bench_phase(ph, iters=200)

    # the optimizer's state (theta, m, v, G: 27 MB) stays L2-resident between back-to-back launches;
    # the same kernel with L2 flushed before every launch (a 512 MB write on the stream) is its DRAM
    # figure (the round itself runs it warm: the state is touched every step)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    cold = []
    for i in range(21):
        flush.fill_(i & 0xff)
        cold.append(g.bench_phase("apply", iters=1))
    apply_cold_us = float(np.median(cold[1:]))
    del flush

    peaks = read_peaks()
    P = g.P
    n_msg = L if args.ps_mode == "per_message" else 1
    # the library's small-batch conv tower (tower.cuh): bf16, 2B <= SMs, not disabled
    tower = (args.math == "bf16" and os.environ.get("GORILA_TOWER", "1") != "0"
             and 2 * args.batch <= torch.cuda.get_device_properties(local_rank).multi_processor_count)
    esz = 2 if args.math == "bf16" else 4
    total_prof = sum(phases.values())
    per_launch_ms = {p: v / max(n_prof, 1) for p, v in phases.items()}
    iso_ms = {p: v / 1000.0 for p, v in iso.items()}
    dom = max(iso_ms, key=lambda p: iso_ms[p])

    def roof(p):
        w = phase_work(p, args.batch, args.n_actions, P, esz, n_msg, tower)
        if w is None or iso_ms.get(p, 0.0) <= 0.0:
            return None
        bound, amount = w
        t = iso_ms[p] / 1000.0
        if bound == "tensor":
            ach = amount / t / 1e12
            # the phase is timed alone, re-launched back to back: the burst peak (B200_PROFILING.md);
            # fp32 check mode runs the SIMT engine (no tensor cores): the bf16 peak / 16 as a marker
            peak = peaks["tensor_burst"] if args.math == "bf16" else peaks["tensor_burst"] / 16
            unit = "TFLOP/s"
        else:
            ach = amount / t / 1e9
            peak = peaks["hbm"]
            unit = "GB/s"
        return {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                "algorithmic_per_launch": amount, "ms_per_launch": iso_ms[p]}

    dom_roof = roof(dom)
    if dom_roof is None:  # dominant phase without an algorithmic model: report the biggest modelled one
        modelled = [p for p in iso_ms if phase_work(p, args.batch, args.n_actions, P, esz, n_msg, tower)]
        dom = max(modelled, key=lambda p: iso_ms[p])
        dom_roof = roof(dom)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.math, {}).get(dom)
        except Exception:
            traffic = None

    if rank == 0:
        clocks = clk.summary()
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16" if args.math == "bf16" else "f32", "data": "synthetic",
            "frames_per_s": value * args.batch,
            "config": config_dict(args, world),
            "gpu_launches": int(launches),
            "timed_region_versions": {"V_before": int(V0), "V_after": int(V1), "last_target_sync_before": int(sync0),
                                      "last_target_sync_after": int(sync1),
                                      "target_syncs": int((V1 - sync0) // args.target_period) if V1 > sync0 else 0},
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 7056 + 1 + 4 + 1,
                    "d2h_bytes_per_step": 48 + 24 + 1,
                    "note": "per step: replay_insert of 1 new transition from pinned host memory (library "
                            "staging ring, read by the scatter kernel over the bus; no stream sync), "
                            "gorila_round_post (learner_step + ps_apply_shard + sync_target as one graph whose last "
                            "node stores the learner info, round info and sync flag into the library's pinned result "
                            "ring), read with gorila_round_fetch one step later (while the next round runs); "
                            f"{args.warmup} untimed warm-up steps of the same loop, {args.e2e_steps} timed"},
            "roofline": {"kernel": dom, "bound": dom_roof["bound"], "achieved": dom_roof["achieved"],
                         "peak": dom_roof["peak"], "unit": dom_roof["unit"], "frac": dom_roof["frac"],
                         "traffic": traffic, "peak_src": peaks["src"],
                         "share_of_step": iso_ms[dom] / (ms / args.steps),
                         "timing": "kernel re-launched back to back on its stream (CUDA events, warm L2, PDL), "
                                   "gorila_bench_phase; share = that time / device ms per step",
                         "ms_per_launch": dom_roof["ms_per_launch"],
                         "algorithmic_per_launch": dom_roof["algorithmic_per_launch"]},
            "apply_dram_cold": {"us_per_launch": apply_cold_us,
                                "achieved_gbs": phase_work("apply", args.batch, args.n_actions, P, esz, n_msg)[1]
                                / (apply_cold_us * 1e-6) / 1e9,
                                "peak_gbs": peaks["hbm"],
                                "note": "k_apply with L2 flushed before each launch (event-timed, median of 20); "
                                        "phase_rooflines.apply is the same kernel back to back with its 27 MB state "
                                        "L2-resident, as inside the training loop"},
            "phases_ms_per_step": {p: v for p, v in per_launch_ms.items() if v > 0},
            "phases_isolated_us": iso,
            "phase_rooflines": {p: roof(p) for p in phases if roof(p) is not None},
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args, args.cpu_seconds)
            out["c1_seconds"] = c1_timing(gpu_c1_seconds)
        print(json.dumps(out), file=json_out, flush=True)
    g.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
