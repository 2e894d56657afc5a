"""paper_1811_00901_b200 — B200-native spin-image engine (arXiv 1811.00901 hot path).

The product is libspin.so (include/spin.h): hand-written sm_100a kernels behind a
C ABI.  `spin` is the ctypes binding with the same names.  Importing this package
loads libspin.so and fails loudly if it is missing (no CPU fallback).
"""
from .spin import (  # noqa: F401
    BILINEAR, BRUTE, CELLS, F_FLOOR_BINS, F_LITERAL_HALF_WIDTH, F_NO_FAST_CERT, F_NO_SORT, FAC,
    GSS, LIB_PATH, NEAREST, F_SUPPORT_LAST, NO_SUPPORT, SS, STATIC, SpinEngine, SpinError, abi_version,
    chunk_sequence, cos_from_degrees, default_P, generate, region_radius,
)
