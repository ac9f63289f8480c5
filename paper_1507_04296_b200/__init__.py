"""B200-native Gorila DQN learner update (Nair et al. 2015, arXiv:1507.04296).

The product is the C-ABI library ``libgorila.so`` (include/gorila.h, sources in
``csrc/``); ``gorila`` is its thin ctypes binding.
"""
from .gorila import (Config, Gorila, GorilaError, LearnerInfo, RoundInfo, EXPORTS, load,  # noqa: F401
                     param_count, nccl_unique_id, phase_names)
