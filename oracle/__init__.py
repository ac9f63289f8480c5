"""CPU oracle for the Gorila DQN learner update (Nair et al. 2015, arXiv:1507.04296).

TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything under
``oracle/``. It shares no code with ``paper_1507_04296_b200`` (the CUDA
path); the only module both use is ``synth`` (seeded input definitions,
none of the method's arithmetic).

Pins: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against something other than itself (Philox
known-answer vectors, closed forms, finite differences, torch CPU library
routines, brute force, SPEC worked examples). The whole learner update as a
composition has no worked example in the paper: "parity unpinned" for the
composition as such (its parts are pinned) — see DESIGN.md.
"""
from .gorila_oracle import *  # noqa: F401,F403
