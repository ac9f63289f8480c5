"""NEXT row f3 on the GPU: gorila_act (batched epsilon-greedy acting on the latest theta^+ replica)
against the oracle's O.act on the same states and Philox draws (Alg.1)."""
import numpy as np
import pytest

import oracle as O
from gpu_util import TOL, make_pair, rel_inf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("math", ["fp32", "bf16"])
def test_f3_epsilon_greedy_acting_parity(math):
    nA, B = 6, 32
    g, orc = make_pair(nA=nA, B=B, C=3000, n_insert=3000, math=math)
    ids = np.array([0], np.int32)
    for k in range(3):  # move theta away from theta0
        g.round(ids, k)
    th = g.get_state()[0]
    states = g.replay_sample(0, 7)["s"]  # u8 [B][4][84][84]
    mode = "bf16" if math == "bf16" else "exact"
    tol = TOL[math]["q"]
    for n, step, eps_final in [(B, 0, 0.1), (B, 500_000, 0.1), (17, 2_000_000, 0.1), (B, 10, 0.0)]:
        a_gpu, q_gpu = g.act(states[:n], step, actor_id=3, eps_final=eps_final, anneal_steps=1_000_000)
        a_ref, Q = O.act(th, states[:n], nA, mode, step, 3, eps_final, 1_000_000, 1507)
        assert rel_inf(q_gpu, Q) <= tol, (step, rel_inf(q_gpu, Q))
        eps = O.epsilon(step, eps_final, 1_000_000)
        for i, (x0, x1) in enumerate(O.act_draws(n, 3, step, 1507)):
            if float(x0) < eps * 4294967296.0:  # exploration: integer-exact
                assert a_gpu[i] == (x1 * nA) >> 32 == a_ref[i]
                continue
            top = np.argsort(-Q[i], kind="stable")
            gap = Q[i][top[0]] - Q[i][top[1]]
            if gap > 2 * tol * np.max(np.abs(Q[i])):  # an unambiguous argmax
                assert a_gpu[i] == a_ref[i], (step, i, a_gpu[i], a_ref[i], gap)
            else:
                assert a_gpu[i] in (top[0], top[1])
    # device-resident states give the same decisions
    import torch
    dev = torch.from_numpy(states).cuda()
    a_d, q_d = g.act(dev, 10, actor_id=3, eps_final=0.0, anneal_steps=1_000_000)
    a_h, q_h = g.act(states, 10, actor_id=3, eps_final=0.0, anneal_steps=1_000_000)
    assert np.array_equal(a_d, a_h) and np.array_equal(q_d, q_h)
