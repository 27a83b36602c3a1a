"""B200-native Atlas hot path (arXiv 2408.09055): C-ABI library + ctypes binding.

The product is libatlas_b200.so (include/atlas.h).  This package only holds its
sources (csrc/), the in-tree build script and the thin binding (atlas.py).
"""
from .atlas import (C128, C64, AtlasError, Simulator, nccl_unique_id, simulate)  # noqa: F401
