import sys, time, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from gpu_util import make_pair
g, _ = make_pair(nA=6, B=32, C=3000, n_insert=3000, math="bf16", ps_mode="async", optimizer="adagrad")
t = time.time()
for sb in (1, 32):
    t = time.time()
    try:
        print(sb, g.async_run([0], 2, server_blocks=sb), time.time() - t, flush=True)
    except Exception as e:
        print(sb, "ERR", e, time.time() - t, flush=True)
        break
