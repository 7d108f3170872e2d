"""B200-native space-time multigrid (arXiv 1411.0519) -- sm_100a CUDA kernels
behind a C ABI (include/stmg_b200.h); this package holds the kernels
(csrc/), the in-tree build and the Python binding of the C ABI."""
from . import _capi  # noqa: F401

__all__ = ["_capi", "stmg", "build"]
