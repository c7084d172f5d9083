"""CPU oracle for the frame-batched GRU-RNNLM query step -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It is
a ctypes binding of ``oracle/oracle.cpp`` (plain C++, fp64 accumulation,
std::map caches) and shares nothing with ``paper_1801_09866_b200``.

Pins: tests/test_oracle_*.py check it against the paper's worked numbers,
closed forms, special cases that reduce to library routines and brute force
(DESIGN.md "Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

KEY_OFF, KEY_ROUND, KEY_SIGN = 0, 1, 2
CELL_GRU, CELL_GRU_LBR, CELL_RNN = 0, 1, 2
QHIT, SHIT, MISS, INVALID = 0, 1, 2, 255
ALL_SESSIONS = 0xFFFFFFFF

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class OrcConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in (
        "V", "E", "H", "maxent_log2", "N", "key_mode", "round_digits",
        "cache_enabled", "num_sessions", "max_histories", "cell")]


class OrcWeights(ctypes.Structure):
    _fields_ = [(n, _f32p) for n in (
        "emb", "Wz", "Uz", "bz", "Wr", "Ur", "br", "Wh", "Uh", "bh",
        "nce_w", "nce_b", "maxent")]


def build(force: bool = False) -> str:
    """Compile oracle.cpp (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["g++", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
                               "-std=c++17", "-shared", "-fPIC", "-o", _SO, _SRC])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.orc_code_bytes.restype = ctypes.c_uint32
        L.orc_code_bytes.argtypes = [ctypes.c_uint32] * 3
        L.orc_compress.restype = ctypes.c_int
        L.orc_compress.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _f32p, _u8p]
        L.orc_maxent_indices.restype = ctypes.c_uint32
        L.orc_maxent_indices.argtypes = [_u32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.c_uint64, _u64p]
        L.orc_gru.restype = None
        L.orc_gru.argtypes = [ctypes.POINTER(OrcConfig), ctypes.POINTER(OrcWeights), _f32p, _f32p,
                              _f64p, _f32p]
        L.orc_score.restype = ctypes.c_float
        L.orc_score.argtypes = [ctypes.POINTER(OrcConfig), ctypes.POINTER(OrcWeights), _f32p, _u32p,
                                ctypes.c_uint32, ctypes.c_uint32]
        L.orc_create.restype = ctypes.c_void_p
        L.orc_create.argtypes = [ctypes.POINTER(OrcConfig), ctypes.POINTER(OrcWeights),
                                 ctypes.POINTER(ctypes.c_int)]
        L.orc_destroy.restype = None
        L.orc_destroy.argtypes = [ctypes.c_void_p]
        L.orc_reset_session.restype = ctypes.c_int
        L.orc_reset_session.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
        L.orc_query_frame.restype = ctypes.c_int
        L.orc_query_frame.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _u32p, _u32p, _u32p, _f32p,
                                      _u32p, _u8p]
        L.orc_stats.restype = ctypes.c_int
        L.orc_stats.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _u64p]
        L.orc_num_handles.restype = ctypes.c_int
        L.orc_num_handles.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _u32p, _u32p]
        for name in ("orc_read_slots",):
            getattr(L, name).restype = ctypes.c_int
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, _u32p,
                                         _u32p]
        L.orc_read_states.restype = ctypes.c_int
        L.orc_read_states.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, _u32p,
                                      _f32p]
        L.orc_read_ctx.restype = ctypes.c_int
        L.orc_read_ctx.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, _u32p, _u32p,
                                   _u32p]
        L.orc_log_normalizer.restype = ctypes.c_double
        L.orc_log_normalizer.argtypes = [ctypes.POINTER(OrcConfig), ctypes.POINTER(OrcWeights), _f32p,
                                         _u32p, ctypes.c_uint32]
        L.orc_log_normalizer_handles.restype = ctypes.c_int
        L.orc_log_normalizer_handles.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                                 _u32p, _f64p]
        L.orc_overwrite_state.restype = ctypes.c_int
        L.orc_overwrite_state.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, _f32p]
        L.orc_threads.restype = ctypes.c_int
        L.orc_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def threads(n: int = 0) -> int:
    """Host threads of the oracle's per-frame scores / GRUs (n > 0 sets it)."""
    return int(lib().orc_threads(n))


def _p(a, t):
    return a.ctypes.data_as(t)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def make_config(V, E, H, maxent_log2, N, key_mode=KEY_OFF, round_digits=0, cache_enabled=1,
                num_sessions=1, max_histories=1 << 16, cell=CELL_GRU) -> OrcConfig:
    return OrcConfig(V, E, H, maxent_log2, N, key_mode, round_digits, cache_enabled,
                     num_sessions, max_histories, cell)


class _Weights:
    """Keeps the float32 arrays alive while the C side holds their pointers."""

    def __init__(self, weights: dict):
        self.arrays = {k: _f32(v) for k, v in weights.items()}
        self.c = OrcWeights(**{k: _p(self.arrays[k], _f32p) for k, _ in OrcWeights._fields_})


def code_bytes(mode: int, k: int, H: int) -> int:
    return int(lib().orc_code_bytes(mode, k, H))


def compress(h, mode: int, k: int = 0) -> np.ndarray:
    h = _f32(h)
    H = h.shape[-1]
    out = np.zeros(code_bytes(mode, k, H), dtype=np.uint8)
    st = lib().orc_compress(mode, k, H, _p(h, _f32p), _p(out, _u8p))
    if st != 0:
        raise ValueError(f"orc_compress status {st}")
    return out


def maxent_indices(ctx, w: int, N: int, M: int) -> list:
    """ctx most recent LAST."""
    c = _u32(ctx if len(ctx) else [0])
    out = np.zeros(16, dtype=np.uint64)
    K = lib().orc_maxent_indices(_p(c, _u32p), len(ctx), w, N, M, _p(out, _u64p))
    return [int(x) for x in out[:K]]


def gru(cfg: OrcConfig, weights: dict, x, h, fp64: bool = False):
    W = _Weights(weights)
    x, h = _f32(x), _f32(h)
    o64 = np.zeros(cfg.H, dtype=np.float64)
    o32 = np.zeros(cfg.H, dtype=np.float32)
    lib().orc_gru(ctypes.byref(cfg), ctypes.byref(W.c), _p(x, _f32p), _p(h, _f32p),
                  _p(o64, _f64p), _p(o32, _f32p))
    return o64 if fp64 else o32


def score(cfg: OrcConfig, weights: dict, h, ctx, w: int) -> float:
    W = _Weights(weights)
    h = _f32(h)
    c = _u32(ctx if len(ctx) else [0])
    return float(lib().orc_score(ctypes.byref(cfg), ctypes.byref(W.c), _p(h, _f32p),
                                 _p(c, _u32p), len(ctx), w))


def log_normalizer(cfg: OrcConfig, weights: dict, h, ctx) -> float:
    """Exact log sum_v exp(score_v) (fp64) for state h and context (most recent LAST)."""
    W = _Weights(weights)
    h = _f32(h)
    c = _u32(ctx if len(ctx) else [0])
    return float(lib().orc_log_normalizer(ctypes.byref(cfg), ctypes.byref(W.c), _p(h, _f32p),
                                          _p(c, _u32p), len(ctx)))


class Oracle:
    """One oracle engine over ``num_sessions`` utterance streams."""

    def __init__(self, cfg: OrcConfig, weights: dict):
        self.cfg = cfg
        self._w = _Weights(weights)
        st = ctypes.c_int(0)
        self._h = lib().orc_create(ctypes.byref(cfg), ctypes.byref(self._w.c), ctypes.byref(st))
        if not self._h:
            raise ValueError(f"orc_create status {st.value}")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    def reset_session(self, s: int):
        assert lib().orc_reset_session(self._h, s) == 0

    def query_frame(self, session, parent, word):
        s, p, w = _u32(session), _u32(parent), _u32(word)
        n = len(s)
        score_ = np.zeros(n, dtype=np.float32)
        child = np.zeros(n, dtype=np.uint32)
        outc = np.zeros(n, dtype=np.uint8)
        lib().orc_query_frame(self._h, n, _p(s, _u32p), _p(p, _u32p), _p(w, _u32p),
                              _p(score_, _f32p), _p(child, _u32p), _p(outc, _u8p))
        return score_, child, outc

    def stats(self, s: int = ALL_SESSIONS) -> dict:
        out = np.zeros(5, dtype=np.uint64)
        sticky = lib().orc_stats(self._h, s, _p(out, _u64p))
        keys = ("total_queries", "query_hits", "hidden_lookups", "hidden_hits", "gru_computations")
        d = {k: int(v) for k, v in zip(keys, out)}
        d["sticky_error"] = int(sticky)
        return d

    def num_handles(self, s: int):
        h = ctypes.c_uint32(0)
        sl = ctypes.c_uint32(0)
        lib().orc_num_handles(self._h, s, ctypes.byref(h), ctypes.byref(sl))
        return h.value, sl.value

    def read_slots(self, s: int, handles):
        h = _u32(handles)
        out = np.zeros(len(h), dtype=np.uint32)
        lib().orc_read_slots(self._h, s, len(h), _p(h, _u32p), _p(out, _u32p))
        return out

    def read_states(self, s: int, handles):
        h = _u32(handles)
        out = np.zeros((len(h), self.cfg.H), dtype=np.float32)
        lib().orc_read_states(self._h, s, len(h), _p(h, _u32p), _p(out, _f32p))
        return out

    def read_ctx(self, s: int, handles):
        h = _u32(handles)
        ctx = np.zeros((len(h), 7), dtype=np.uint32)
        ln = np.zeros(len(h), dtype=np.uint32)
        lib().orc_read_ctx(self._h, s, len(h), _p(h, _u32p), _p(ctx, _u32p), _p(ln, _u32p))
        return [list(ctx[i, :ln[i]]) for i in range(len(h))]

    def log_normalizer(self, s: int, handles):
        h = _u32(handles)
        out = np.zeros(len(h), dtype=np.float64)
        assert lib().orc_log_normalizer_handles(self._h, s, len(h), _p(h, _u32p), _p(out, _f64p)) == 0
        return out

    def overwrite_state(self, s: int, handle: int, h):
        h = _f32(h)
        assert lib().orc_overwrite_state(self._h, s, handle, _p(h, _f32p)) == 0


def resolve_parents(parent_ref: np.ndarray, child_log: np.ndarray) -> np.ndarray:
    """Workload references -> history handles, from the engine's own outputs."""
    return np.where(parent_ref >= 0, child_log[np.maximum(parent_ref, 0)], 0).astype(np.uint32)


def run_workload(orc: Oracle, wl, frames=None):
    """Run frames of a synth.Workload; returns (score, child, outcome) flat arrays."""
    F = wl.frames if frames is None else frames
    n = F * wl.n_per_frame
    score_ = np.zeros(n, dtype=np.float32)
    child = np.zeros(n, dtype=np.uint32)
    outc = np.zeros(n, dtype=np.uint8)
    for t in range(F):
        sl = wl.frame_slice(t)
        par = resolve_parents(wl.parent_ref[sl], child)
        sc, ch, oc = orc.query_frame(wl.session[sl], par, wl.word[sl])
        score_[sl], child[sl], outc[sl] = sc, ch, oc
    return score_, child, outc
