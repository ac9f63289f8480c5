"""A minimal run for compute-sanitizer: one round in each math mode (B = 8, nA = 4): sampler, conv tower
(bf16) / SIMT GEMMs (fp32), TMA / shifted-window GEMMs, fc5 + TD, backward, reduce, apply, sync."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1507_04296_b200 import Gorila  # noqa: E402

for math in (sys.argv[1:] or ["bf16", "fp32"]):
    g = Gorila(n_actions=4, batch=8, replay_capacity=300, theta0=synth.theta0(4), math=math, target_period=1)
    f = synth.frames(synth.SEED_DATA, 0, 0, 300)
    a, r, d = synth.meta(synth.SEED_DATA, 0, 0, 300, 4)
    g.replay_insert(0, f, a, r, d)
    ids = np.zeros(1, np.int32)
    for k in range(2):
        g.learner_step([0], k)
        g.ps_apply_shard(k)
        g.sync_target([0])
    print(math, "ok", g.get_state()[3], flush=True)
    g.close()
