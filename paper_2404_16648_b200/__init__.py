"""B200-native fp64 dGSEM right-hand side of arXiv 2404.16648's tree-based AMR path.

The product is the C-ABI library libdg (include/dg.h; csrc/ = host runtime +
sm_100a kernels) and this thin binding (dg.py).  Importing the package loads
lib/libdg.so and fails loudly if it is missing; there is no CPU fallback.
"""
from . import dg  # noqa: F401
from .dg import DG, DGError, from_device, to_device  # noqa: F401

__all__ = ["dg", "DG", "DGError", "to_device", "from_device"]
