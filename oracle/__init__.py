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
routines, brute force, SPEC worked examples). The paper prints no worked
example of the whole learner update; the composed round (sample → forward →
TD → backward → RMSProp step) is pinned by a closed form instead: with W1 = 0
every activation is spatially constant and the round reduces to written-out
sums (tests/test_oracle_round_closed_form.py) — see DESIGN.md §3.
"""
from .gorila_oracle import *  # noqa: F401,F403
