"""B200-native frame-batched GRU-RNNLM query step (arXiv 1801.09866 hot path).

The product is librnnlm.so (hand-written sm_100a kernels behind the C ABI of
include/rnnlm.h); this package is its thin binding plus host-side reporting.
"""
from .engine import (ALL, CELL_GRU, CELL_GRU_LBR, CELL_RNN, GRU_AUTO, GRU_GEMV, GRU_TILES, INVALID, KEY_MODES, KEY_OFF,
                     KEY_ROUND, KEY_SIGN, MATH_BF16, MATH_BF16X3, MATH_FP32, MATH_TF32, MATH_TF32X3, MISS, QHIT, RNNLM, SHIT,
                     StepGraph, as_u32, resolve_parents)
from .stats import hit_ratio, redundancy_rate

__all__ = ["RNNLM", "KEY_OFF", "KEY_ROUND", "KEY_SIGN", "KEY_MODES", "MATH_FP32", "MATH_TF32", "MATH_BF16", "MATH_TF32X3", "MATH_BF16X3",
           "QHIT", "SHIT", "MISS", "INVALID", "ALL", "resolve_parents", "as_u32", "CELL_GRU", "CELL_GRU_LBR", "CELL_RNN",
           "redundancy_rate", "hit_ratio", "GRU_AUTO", "GRU_TILES", "GRU_GEMV", "StepGraph"]
