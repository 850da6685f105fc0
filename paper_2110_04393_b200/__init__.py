"""B200-native randomized TT-rounding of sums (arXiv 2110.04393, Alg. 7).

Thin ctypes binding of libttround.so (include/ttround.h): argument marshalling
only — every arithmetic step of the hot path runs in the library's CUDA kernels.
There is no CPU fallback: importing this package raises if the library is
missing, and every call raises ``TTError`` on a non-zero return code.
"""
from ._lib import (  # noqa: F401
    LIB_PATH, TTError, Context, LoopbackGroup, Plan, Sketch, TTResult, SKETCH_ONLY, RANK, TOL,
    FLAG_RANK_CAPPED, FLAG_LEFT_ORTH, FLAG_RIGHT_ORTH, FLAG_ZERO, FLAG_QR_FALLBACK, FLAG_SLAB,
    tt_launch_count, tt_get_nccl_unique_id, load_library,
)
