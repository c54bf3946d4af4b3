"""B200-native (sm_100a) SPLAT sparse-MHSA hot path (arXiv 2407.16847).

The product is the C-ABI library ``libsplat.so`` (include/splat.h); this
package holds its CUDA sources (csrc/), the in-tree build (build.py) and a
thin ctypes binding (splat.py).  Importing the package does not load the
library; the first call does, and fails loudly if it is missing.
"""
from .splat import (Acsr, SplatError, splat_acsr_build, splat_rsddmm, splat_sparse_softmax, splat_rspmm,
                    splat_sparse_mhsa, splat_sparse_mhsa_host)

__all__ = ["Acsr", "SplatError", "splat_acsr_build", "splat_rsddmm", "splat_sparse_softmax", "splat_rspmm",
           "splat_sparse_mhsa", "splat_sparse_mhsa_host"]
