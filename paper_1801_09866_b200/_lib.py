"""ctypes binding of librnnlm.so (include/rnnlm.h).  Argument marshalling only.

Loading fails loudly if the library is missing: there is no CPU or eager
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

_u32p = ctypes.POINTER(ctypes.c_uint32)
_vp = ctypes.c_void_p


class Config(ctypes.Structure):
    _fields_ = [("vocab", ctypes.c_uint32), ("embed", ctypes.c_uint32), ("hidden", ctypes.c_uint32),
                ("maxent_log2", ctypes.c_uint32), ("maxent_order", ctypes.c_uint32),
                ("key_mode", ctypes.c_uint32), ("round_digits", ctypes.c_uint32),
                ("math", ctypes.c_uint32), ("cache_enabled", ctypes.c_uint32),
                ("num_sessions", ctypes.c_uint32), ("max_queries_per_call", ctypes.c_uint32),
                ("max_histories_per_session", ctypes.c_uint32), ("device", ctypes.c_int32),
                ("cell", ctypes.c_uint32), ("max_queries_per_session_call", ctypes.c_uint32),
                ("gru_path", ctypes.c_uint32)]


WEIGHT_NAMES = ("emb", "Wz", "Uz", "bz", "Wr", "Ur", "br", "Wh", "Uh", "bh", "nce_w", "nce_b",
                "maxent")


class Weights(ctypes.Structure):
    _fields_ = [(n, _vp) for n in WEIGHT_NAMES]


class Stats(ctypes.Structure):
    _fields_ = [("total_queries", ctypes.c_uint64), ("query_hits", ctypes.c_uint64),
                ("hidden_lookups", ctypes.c_uint64), ("hidden_hits", ctypes.c_uint64),
                ("gru_computations", ctypes.c_uint64), ("sticky_error", ctypes.c_int32),
                ("pad_", ctypes.c_int32)]


class Timing(ctypes.Structure):
    _fields_ = [("ms_cache", ctypes.c_double), ("ms_score", ctypes.c_double),
                ("ms_gru", ctypes.c_double), ("ms_encode", ctypes.c_double),
                ("ms_final", ctypes.c_double), ("calls", ctypes.c_uint64),
                ("launches", ctypes.c_uint64), ("ms_gru_gather", ctypes.c_double),
                ("ms_gru_phase1", ctypes.c_double), ("ms_gru_phase2", ctypes.c_double),
                ("ms_fused", ctypes.c_double)]


# name -> (restype, argtypes); every symbol include/rnnlm.h declares
SIGNATURES = {
    "rnnlm_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(Weights),
                                    ctypes.POINTER(_vp)]),
    "rnnlm_destroy": (None, [_vp]),
    "rnnlm_reset_session": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp]),
    "rnnlm_query_batch": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rnnlm_cache_stats": (ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.POINTER(Stats)]),
    "rnnlm_read_states": (ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp, _vp]),
    "rnnlm_read_slots": (ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp, _vp]),
    "rnnlm_read_codes": (ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp, _vp]),
    "rnnlm_encode_states": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp, _vp, _vp]),
    "rnnlm_log_normalizer": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp, _vp, _vp, _vp]),
    "rnnlm_results_ready": (ctypes.c_int, [_vp, _vp]),
    "rnnlm_maxent_indices": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp, _vp, _vp, _vp, _vp]),
    "rnnlm_code_bytes": (ctypes.c_uint32, [_vp]),
    "rnnlm_resolve_parents": (ctypes.c_int, [ctypes.c_uint32, _vp, _vp, _vp, _vp]),
    "rnnlm_set_timing": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rnnlm_get_timing": (ctypes.c_int, [_vp, ctypes.POINTER(Timing), ctypes.c_int]),
    "rnnlm_launch_count": (ctypes.c_uint64, [_vp]),
    "rnnlm_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "rnnlm_abi_version": (ctypes.c_int, []),
    "rnnlm_graph_create": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                          ctypes.POINTER(_vp)]),
    "rnnlm_graph_launch": (ctypes.c_int, [_vp, _vp]),
    "rnnlm_graph_destroy": (None, [_vp]),
    "rnnlm_tf32x3_products": (ctypes.c_double, [_vp]),
}

_lib = None


def library_path() -> str:
    # RNNLM_LIBRARY: another in-tree build of the same ABI (A/B experiments only)
    return os.environ.get("RNNLM_LIBRARY") or _build.SO


def load():
    """Load librnnlm.so (RuntimeError if it has not been built)."""
    global _lib
    if _lib is None:
        path = library_path()
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: run `python -m paper_1801_09866_b200.build` "
                               "(or __graft_entry__.build()); there is no fallback path")
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RnnlmError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        msg = load().rnnlm_status_string(status).decode()
        super().__init__(f"{what}: {msg} (status {status})" if what else msg)
        self.status = status


def check(status: int, what: str = ""):
    if status != 0:
        raise RnnlmError(status, what)
