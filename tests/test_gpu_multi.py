"""Multi-rank parity of the sharded parameter server: tools/multi_gpu_check.py under torchrun.

Two launch shapes, the same data path (k_apply_p2p / k_peer_wait / k_replay_barrier over peer
memory, "split disjointly", Alg.1 P:116 / P:129):
* ipc: a gloo process group and every rank on cuda:0 -- several ranks share one GPU, the CUDA IPC
  records of their workspaces exchanged over gloo (gorila_peer_connect). Runs on a 1-GPU box, up to
  the exchange's maximum of 8 ranks (the GPU time-slices the ranks' contexts; the exchange's flag
  waits make progress across those slices).
* nccl: one rank per GPU (>= 2 GPUs), the library's NCCL communicator bootstraps the mappings.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

MODES = {"aggregate": {}, "per_message_f1": {"PS_MODE": "per_message", "L_LOCAL": "2"},
         "global_replay_f4": {"REPLAY": "global"}}


def _run(n, env, timeout=900):
    env = dict(os.environ, **env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + (os.getpid() % 300) + 7 * n),
           os.path.join(ROOT, "tools", "multi_gpu_check.py")]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0 and "MULTI-GPU CHECK OK" in out.stdout, out.stdout[-4000:] + out.stderr[-3000:]
    return out.stdout


@pytest.mark.parametrize("math", ["fp32", "bf16"])
@pytest.mark.parametrize("mode", list(MODES))
def test_sharded_ps_two_ranks_one_gpu(math, mode):
    print(_run(2, dict(MATH=math, ROUNDS="4", BOOTSTRAP="ipc", CUDA_VISIBLE_DEVICES=_first_gpu(), **MODES[mode])))


def test_large_batch_global_replay_two_ranks_one_gpu():
    """B = 80 (the large-batch path: conv1 bulk-copies its frames straight from the replay rings) with
    global replay (f4): half of the draws' frames live in the other rank's ring, read through the peer
    mapping by the same bulk copies."""
    print(_run(2, dict(MATH="bf16", ROUNDS="3", BOOTSTRAP="ipc", BATCH="80", REPLAY="global",
                       CUDA_VISIBLE_DEVICES=_first_gpu())))


@pytest.mark.parametrize("n", [4, 8])
def test_sharded_ps_many_ranks_one_gpu(n):
    """W = 4 and the exchange's maximum W = 8 (MAX_W): eight shards, eight owners."""
    print(_run(n, dict(MATH="bf16", ROUNDS="3", BOOTSTRAP="ipc", CUDA_VISIBLE_DEVICES=_first_gpu()), timeout=1200))


@pytest.mark.parametrize("math", ["fp32", "bf16"])
@pytest.mark.parametrize("mode", list(MODES))
def test_sharded_ps_one_rank_per_gpu_nccl(math, mode):
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (the one-GPU shape is covered by the ipc tests above)")
    print(_run(min(n, 4), dict(MATH=math, ROUNDS="4", BOOTSTRAP="nccl", **MODES[mode])))


def _first_gpu():
    v = os.environ.get("CUDA_VISIBLE_DEVICES")
    return v.split(",")[0] if v else "0"


@pytest.mark.parametrize("n", [2, 4])
def test_async_ps_several_ranks_one_gpu(n):
    """NEXT row f2 across ranks: every rank's shard server applies every rank's messages as they arrive
    (tools/async_check.py: counts add up on every shard, theta^+ agrees across ranks)."""
    env = dict(os.environ, BOOTSTRAP="ipc", CUDA_VISIBLE_DEVICES=_first_gpu(), STEPS="8")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29950 + (os.getpid() % 40) + 3 * n),
           os.path.join(ROOT, "tools", "async_check.py")]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "ASYNC CHECK OK" in out.stdout, out.stdout[-4000:] + out.stderr[-3000:]
    print(out.stdout)
