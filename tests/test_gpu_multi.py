"""Multi-GPU parity (>= 2 GPUs): tools/multi_gpu_check.py under torchrun, one rank per GPU."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("math", ["fp32", "bf16"])
@pytest.mark.parametrize("mode", [{}, {"PS_MODE": "per_message"}, {"REPLAY": "global"}],
                         ids=["aggregate", "per_message_f1", "global_replay_f4"])
def test_sharded_ps_over_nccl_matches_oracle(math, mode):
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 4)
    env = dict(os.environ, MATH=math, ROUNDS="4", **mode)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + (os.getpid() % 500)),
           os.path.join(ROOT, "tools", "multi_gpu_check.py")]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "MULTI-GPU CHECK OK" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]
