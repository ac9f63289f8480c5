"""NEXT row f3 (acting): the oracle's epsilon-greedy rule against closed forms and statistics
(Alg.1; P:187 linear anneal)."""
import numpy as np

import oracle as O
import synth


def test_epsilon_linear_anneal_closed_form():
    assert O.epsilon(0, 0.1, 1_000_000) == 1.0
    assert O.epsilon(1_000_000, 0.1, 1_000_000) == 0.1
    assert O.epsilon(5_000_000, 0.1, 1_000_000) == 0.1
    assert abs(O.epsilon(500_000, 0.1, 1_000_000) - 0.55) < 1e-15
    assert abs(O.epsilon(250_000, 0.0, 1_000_000) - 0.75) < 1e-15


def _zero_net(nA, b5):
    th = np.zeros(O.param_count(nA))
    p = O.unflatten(th, nA)
    p["b5"][:] = b5
    return th


def test_greedy_is_lowest_index_argmax():
    """Zero weights: Q(s, .) = b5 for every s; ties go to the lowest index (epsilon = 0)."""
    nA = 4
    th = _zero_net(nA, [0.5, 0.9, 0.9, 0.1])
    s = synth.frames(synth.SEED_DATA, 0, 0, 12)[:8].reshape(2, 4, 84, 84)
    for mode in ("exact", "bf16"):
        a, Q = O.act(th, s, nA, mode, 10, 0, 0.0, 1, 1507)
        assert np.array_equal(a, [1, 1]) and np.allclose(Q, [[0.5, 0.9, 0.9, 0.1]] * 2)


def test_full_exploration_uses_the_philox_draw_and_is_uniform():
    nA, n = 6, 3000
    th = _zero_net(nA, [0.0] * nA)
    draws = O.act_draws(n, 7, 0, 1507)
    # epsilon = 1 at step 0: every action is floor(x1 * nA / 2^32)
    s = np.zeros((4, 4, 84, 84), np.uint8)
    a, _ = O.act(th, s, nA, "exact", 0, 7, 0.1, 1_000_000, 1507)
    assert list(a) == [(x1 * nA) >> 32 for _, x1 in draws[:4]]
    counts = np.bincount([(x1 * nA) >> 32 for _, x1 in draws], minlength=nA)
    chi2 = float(((counts - n / nA) ** 2 / (n / nA)).sum())
    assert chi2 < 20.5  # 5 dof, p ~ 0.001
    assert counts.min() > 0


def test_exploration_rate_matches_epsilon():
    n = 4000
    draws = O.act_draws(n, 3, 500_000, 1507)
    eps = O.epsilon(500_000, 0.1, 1_000_000)  # 0.55
    k = sum(1 for x0, _ in draws if float(x0) < eps * 4294967296.0)
    sd = np.sqrt(n * eps * (1 - eps))
    assert abs(k - n * eps) < 4 * sd
