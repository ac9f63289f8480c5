"""Per-layer check of the bf16 forward convolutions on the GPU's own inputs (diagnostics).

Runs the C1 teacher-forced rounds; after round K fetches s, a1, a2, a3 of the learner step
and recomputes each conv layer in fp64 from the GPU's own (bf16) input, then rounds to bf16:
elements differing by more than one bf16 ulp, and their pre-activation magnitude, are listed.
usage: python tools/diag_conv.py [round]
"""
import sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O
from gpu_util import make_pair, teacher_force, run_round_both

K = int(sys.argv[1]) if len(sys.argv) > 1 else 7


def bf16(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


g, orc = make_pair(nA=4, B=32, C=10_000, n_insert=10_000, math="bf16", target_period=5, outlier_warmup=2)
for k in range(K + 1):
    teacher_force(g, orc)
    th = g.get_state()[0].astype(np.float64)
    gpu, res = run_round_both(g, orc, k, [0])
p = O.unflatten(th, 4)
s, a1, a2, a3 = (g.get_activation(n).astype(np.float64) for n in ("s", "a1", "a2", "a3"))
wb = {k2: bf16(v).astype(np.float64) for k2, v in p.items()}
nchw = lambda t: np.ascontiguousarray(t.transpose(0, 3, 1, 2))
for name, x, w, b, stride, y, scale in (("conv1", s, "W1", "b1", 4, a1, 1 / 255.0),
                                        ("conv2", a1, "W2", "b2", 2, a2, 1.0),
                                        ("conv3", a2, "W3", "b3", 1, a3, 1.0)):
    # conv1 weights see the raw bytes; 1/255 scales the accumulated sum (as the kernel does)
    z = O.conv2d_fwd(nchw(x), wb[w], np.zeros_like(p[b]), stride) * scale
    z = z.transpose(0, 2, 3, 1) + p[b]
    ref = bf16(np.maximum(z, 0)).astype(np.float64)
    ulp = np.maximum(np.abs(ref), 1e-30) * 2.0 ** -7
    bad = np.abs(y - ref) > 1.01 * ulp
    print(name, "elements", y.size, "beyond 1 ulp", int(bad.sum()), "max |z| there",
          float(np.abs(z[bad]).max()) if bad.any() else 0, "max |z|", float(np.abs(z).max()))
    if bad.any():
        idx = np.argwhere(bad)[:12]
        for i in idx:
            t = tuple(i)
            print("   ", t, "gpu", y[t], "ref", ref[t], "z", z[t])
