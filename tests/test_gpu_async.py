"""NEXT row f2: the asynchronous parameter server (ps_mode "async", include/gorila.h gorila_async_run).

Asynchronous SGD has no deterministic result to compare with an oracle (throughput-only);
what is checked:
* one learner: each step fetches only after its previous message was applied (the learner waits for its
  own gradient buffer), so the asynchronous run is exactly the per-message deterministic mode (f1) with
  one learner -- theta, m, v, V and the target net must match it bit for bit (and f1 is oracle-checked);
* several learners: real staleness appears (a learner fetches while others' messages are in flight); the
  counts must add up (sent + rejected = steps, fresh + stale = sent, V = fresh), the observed delays must
  be consistent with the discard threshold, and the deterministic entry points are refused.
"""
import numpy as np
import pytest

from gpu_util import make_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("math", ["bf16", "fp32"])
def test_async_single_learner_equals_per_message_mode(math):
    kw = dict(nA=6, B=32, C=3000, n_insert=3000, math=math, optimizer="adagrad", lr=1e-3, ada_eps=1e-6,
              target_period=3, outlier_warmup=2)
    ga, _ = make_pair(ps_mode="async", **kw)
    gm, _ = make_pair(ps_mode="per_message", **kw)
    K = 7
    st = ga.async_run([0], K)
    for k in range(K):
        gm.round(np.array([0], np.int32), k)
    assert st["steps"] == K and st["sent"] + st["rejected"] == K and st["fresh"] + st["stale"] == st["sent"]
    assert st["max_delay"] == 0 and st["version_after"] == st["fresh"]
    ta, ma, va, Va = ga.get_state()
    tm, mm, vm, Vm = gm.get_state()
    assert Va == Vm == st["fresh"]
    assert np.array_equal(ta, tm) and np.array_equal(ma, mm) and np.array_equal(va, vm)
    assert np.array_equal(ga.get_learner_state(0)[0], gm.get_learner_state(0)[0])


def test_async_several_learners_counts_and_staleness():
    from paper_1507_04296_b200 import GorilaError
    L, K, max_delay = 4, 12, 1
    g, _ = make_pair(nA=6, B=32, C=3000, n_insert=3000, math="bf16", L=L, ps_mode="async",
                     max_staleness=max_delay, target_period=5, outlier_warmup=2)
    th0 = g.get_state()[0]
    st = g.async_run(list(range(L)), K, server_blocks=16)
    assert st["steps"] == K * L
    assert st["sent"] + st["rejected"] == K * L
    assert st["fresh"] + st["stale"] == st["sent"] and st["version_after"] == st["fresh"]  # from V = 0
    assert st["fresh"] >= 1 and st["mean_delay"] <= st["max_delay"]
    # a message is discarded iff its delay exceeded the threshold: with stale ones, delays above it occurred
    assert (st["stale"] > 0) == (st["max_delay"] > max_delay)
    th1, _, _, V = g.get_state()
    assert V == st["fresh"] and np.all(np.isfinite(th1)) and not np.array_equal(th0, th1)
    with pytest.raises(GorilaError):
        g.learner_step([0, 1, 2, 3], 0)
    # a second run continues from the live state
    st2 = g.async_run(list(range(L)), 3, round0=K)
    assert g.get_state()[3] == st2["version_after"] == st["fresh"] + st2["fresh"]
    print("async counts:", st, st2)
