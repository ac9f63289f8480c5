"""C-ABI checks that need no GPU: the library builds, loads, exports every symbol
include/gorila.h declares, and the ctypes structs match the C layouts."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gorila.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"GORILA_API\s+[\w\s\*]+?\b(\w+)\s*\(", src)))


def test_header_declares_the_six_paper_calls():
    names = _declared()
    for n in ("gorila_init", "replay_insert", "replay_sample", "learner_step", "ps_apply_shard", "sync_target"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1507_04296_b200 import gorila as G
    lib = G.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(G.EXPORTS) == _declared()
    # pure host functions work without a GPU
    assert G.param_count(18) == 1_693_362 and G.param_count(4) == 1_686_180


def test_ctypes_struct_layouts_match_c():
    from paper_1507_04296_b200 import gorila as G
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "gorila.h"
int main(void) {
  printf("%zu %zu %zu\n", sizeof(gorila_config), sizeof(gorila_learner_info), sizeof(gorila_round_info));
  printf("%zu %zu %zu %zu %zu\n", offsetof(gorila_config, replay_capacity), offsetof(gorila_config, workspace_bytes),
         offsetof(gorila_config, target_period), offsetof(gorila_config, outlier_beta), offsetof(gorila_config, theta0));
  printf("%zu %zu\n", offsetof(gorila_learner_info, base_version), offsetof(gorila_learner_info, accepted));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-std=c11", "-I" + os.path.join(ROOT, "include"), c, "-o", exe])
        out = subprocess.check_output([exe]).decode().split()
    vals = [int(x) for x in out]
    assert vals[:3] == [ctypes.sizeof(G.Config), ctypes.sizeof(G.LearnerInfo), ctypes.sizeof(G.RoundInfo)]
    assert vals[3:8] == [G.Config.replay_capacity.offset, G.Config.workspace_bytes.offset,
                         G.Config.target_period.offset, G.Config.outlier_beta.offset, G.Config.theta0.offset]
    assert vals[8:] == [G.LearnerInfo.base_version.offset, G.LearnerInfo.accepted.offset]


def test_product_package_does_not_touch_the_oracle():
    pkg = os.path.join(ROOT, "paper_1507_04296_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|oracle/|liboracle)", txt), f


def test_sass_contains_tcgen05_and_tmem_loads():
    from paper_1507_04296_b200 import _build
    _build.build()
    try:
        sass = subprocess.check_output(["cuobjdump", "-sass", _build.SO], stderr=subprocess.STDOUT).decode()
    except FileNotFoundError:
        pytest.skip("cuobjdump not available")
    assert "UTCHMMA" in sass and "LDTM" in sass


def _base_cfg(G, theta):
    c = G.Config()
    c.n_actions, c.batch, c.gamma, c.replay_capacity = 18, 32, 0.99, 1000
    c.n_learners_local, c.learner_id_base, c.rank, c.world = 1, 0, 0, 1
    c.optimizer, c.lr, c.rms_rho, c.rms_eps, c.ada_eps = G.GORILA_OPT_RMSPROP, 2.5e-4, 0.95, 0.01, 1e-8
    c.target_period, c.max_staleness, c.history = 100, -1, 2
    c.math, c.ps_mode, c.replay_mode = G.GORILA_MATH_FP32, 0, 0
    c.theta0 = theta.ctypes.data
    c.workspace = None  # validated last: the only error a valid config reaches without a GPU
    return c


@pytest.mark.parametrize("field,value,msg", [
    ("n_actions", 0, "n_actions"), ("n_actions", 33, "n_actions"),   # P:182 one output per action, <= 32 (R5)
    ("batch", 0, "batch"), ("batch", 4097, "batch"),
    ("replay_capacity", 1, "replay_capacity"), ("n_learners_local", 0, "n_learners_local"),
    ("world", 0, "rank/world"), ("rank", 1, "rank/world"), ("math", 1, "math"),
    ("history", 0, "history"), ("history", 65, "history"), ("target_period", 0, "target_period"),
    ("ps_mode", 3, "ps_mode"), ("ps_mode", -1, "ps_mode"), ("replay_mode", 2, "replay_mode"), ("theta0", None, "theta0"),
    (None, None, "workspace"),
])
def test_init_rejects_invalid_config_before_any_cuda_call(field, value, msg):
    """Error behaviour of gorila_init (include/gorila.h): E_INVALID, a message naming the field,
    *out set to NULL — all decided before the library touches the device."""
    import numpy as np
    from paper_1507_04296_b200 import gorila as G
    lib = G.load()
    theta = np.zeros(lib.gorila_param_count(18), np.float32)
    c = _base_cfg(G, theta)
    if field is not None:
        setattr(c, field, value)
    out = ctypes.c_void_p(1)
    st = lib.gorila_init(ctypes.byref(c), ctypes.byref(out))
    assert G.STATUS[st] == "E_INVALID"
    assert msg in lib.gorila_last_error().decode()
    assert out.value is None


def test_calls_on_a_null_context_fail_cleanly():
    from paper_1507_04296_b200 import gorila as G
    lib = G.load()
    assert G.STATUS[lib.gorila_init(None, None)] == "E_INVALID"
    assert G.STATUS[lib.replay_insert(None, 0, 1, None, None, None, None, 0)] == "E_INVALID"
    assert G.STATUS[lib.learner_step(None, None, 1, 0, None, None)] == "E_INVALID"
    assert G.STATUS[lib.ps_apply_shard(None, 0, None)] == "E_INVALID"
    assert "null" in lib.gorila_last_error().decode()
