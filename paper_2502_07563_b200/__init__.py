"""B200-native LASP-2 / LASP-2H sequence-parallel attention (arXiv 2502.07563).

Drop-in for the reference laspsim hot path (lasp2, standard_sp): same entry
points and BHND layouts over torch CUDA tensors, computed by hand-written
sm_100a kernels behind the C ABI in include/lasp2_b200.h.
"""
__version__ = "0.1.0"

from . import comm, datagen, lasp2, ops, shards, standard_sp  # noqa: F401
