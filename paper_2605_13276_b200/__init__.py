"""paper_2605_13276_b200 -- B200-native hot path of D-VLA's data plane.

Drop-in for the reference `dvla` package's learner, rollout-head and
weight-sync interfaces (reference pkg/src/dvla/{grpo,policy,core,planes,
pools,runtime}.py), implemented as sm_100a CUDA kernels behind the C-ABI in
include/dvla_b200.h (libdvla_b200.so, built in-tree by `build.py`).

Submodules import lazily so that host-only pieces (config types, the arena
bookkeeping, wire frames) work in a CPU container; every compute call needs
the CUDA library and a B200 -- there is no CPU fallback.
"""

__version__ = "0.1.0"
