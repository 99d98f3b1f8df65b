"""B200-native IRLS s-t min-cut hot path (Zhu & Gleich, arXiv 1501.03105).

The product is libirls_mincut.so (C ABI in include/irls_mincut.h, CUDA kernels
for sm_100a in csrc/); ``irls`` is its ctypes binding.
"""
from .irls import (IRLS_CONTINUE, IRLS_FROM_SCRATCH, IRLS_LOOP_GRAPH, IRLS_LOOP_HOST,  # noqa: F401
                   IRLS_NORM_PRECONDITIONED, IRLS_NORM_UNPRECONDITIONED, IrlsError, MinCut, comm_desc, lib,
                   options)
