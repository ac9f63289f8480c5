"""CPU checks of the parity protocol's teacher forcing (R30): the oracle's pre-activation
output is consistent with its activations, and teacher_forced_acts takes the GPU's decision only
where it is ambiguous."""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_util import ACT_LAYERS, BAND, teacher_forced_acts


@pytest.mark.parametrize("mode", ["exact", "bf16"])
def test_oracle_preactivations_match_its_activations(mode):
    """a_l = ReLU(z_l) (rounded to bf16 for a1..a3 in BF16 mode, R16): the exported z is the value
    the oracle's ReLU decided on, and exporting it changes nothing."""
    nA = 4
    th = synth.theta0(nA)
    s = np.random.default_rng(3).integers(0, 256, (3, 4, 84, 84), dtype=np.uint8)
    Q, acts, zs = O.qnet_forward(th, s, nA, mode, want_z=True)
    Q2, acts2 = O.qnet_forward(th, s, nA, mode)
    assert np.array_equal(Q, Q2) and np.array_equal(acts, acts2)
    h = np.maximum(zs, 0.0)
    if mode == "bf16":
        n3 = sum(int(np.prod(shp)) for _, shp in ACT_LAYERS[:3])
        h[:, :n3] = np.vectorize(O.round_bf16)(h[:, :n3])
    assert np.array_equal(h, acts)
    assert (zs < 0).any() and (zs > 0).any()


def _fake(B=2, seed=0):
    rng = np.random.default_rng(seed)
    n = sum(int(np.prod(shp)) for _, shp in ACT_LAYERS)
    zs = rng.normal(size=(B, n))
    return zs, np.maximum(zs, 0.0)


def test_forcing_takes_the_gpu_decision_only_where_ambiguous():
    zs, acts = _fake()
    zs[0, 5] = -1e-7 * np.abs(zs[:, :12800]).max()   # a1 element just below 0
    acts[0, 5] = 0.0
    gpu = acts.copy()
    gpu[0, 5] = 2e-7                                    # the GPU's sum landed just above 0
    log = []
    out = teacher_forced_acts(gpu, acts, zs, "fp32", log)
    assert out[0, 5] == gpu[0, 5] and log == [{"a1": 1, "a2": 0, "a3": 0, "a4": 0}]
    mask = np.ones(acts.shape, bool)
    mask[0, 5] = False
    assert np.array_equal(out[mask], acts[mask])       # nothing else moves


def test_forcing_rejects_a_clear_decision():
    zs, acts = _fake()
    i = int(np.argmax(zs[0, :12800]))                   # the layer's largest pre-activation
    gpu = acts.copy()
    gpu[0, i] = 0.0                                     # the GPU switched it off: a real error
    with pytest.raises(AssertionError):
        teacher_forced_acts(gpu, acts, zs, "bf16")


def test_forcing_rejects_too_many_flips():
    zs, acts = _fake()
    n1 = 12800
    zs[:, :n1] *= 1e-9                                  # make the whole first layer "ambiguous"
    zs[0, n1 - 1] = 1.0
    acts = np.maximum(zs, 0.0)
    gpu = acts.copy()
    flip = np.flatnonzero(acts[1, :n1] > 0)[:50]        # 50 flips > 1e-4 of 25600 elements
    gpu[1, flip] = 0.0
    assert BAND["bf16"] > 0
    with pytest.raises(AssertionError):
        teacher_forced_acts(gpu, acts, zs, "bf16")
