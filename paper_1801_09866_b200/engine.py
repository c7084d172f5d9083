"""Thin Python binding of the C ABI (include/rnnlm.h) over torch device memory.

Every step of the query path runs in librnnlm.so's kernels; this module only
marshals pointers, sizes and the current CUDA stream.  Names follow the C ABI.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import Config, Stats, Timing, Weights, check

KEY_OFF, KEY_ROUND, KEY_SIGN = 0, 1, 2
MATH_FP32, MATH_TF32, MATH_BF16, MATH_TF32X3, MATH_BF16X3 = 0, 1, 2, 3, 4
CELL_GRU, CELL_GRU_LBR, CELL_RNN = 0, 1, 2  # rnnlm_cell
GRU_AUTO, GRU_TILES, GRU_GEMV = 0, 1, 2  # rnnlm_gru_path
QHIT, SHIT, MISS, INVALID = 0, 1, 2, 255
ALL = 0xFFFFFFFF

KEY_MODES = {"off": (KEY_OFF, 0), "sign": (KEY_SIGN, 0), "round:1": (KEY_ROUND, 1),
             "round:2": (KEY_ROUND, 2), "round:3": (KEY_ROUND, 3), "round:4": (KEY_ROUND, 4)}


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class RNNLM:
    """One engine (rnnlm_t) on one CUDA device over ``num_sessions`` streams."""

    def __init__(self, weights: dict, *, vocab: int, embed: int, hidden: int, maxent_log2: int,
                 maxent_order: int, key_mode: int = KEY_OFF, round_digits: int = 0,
                 math: int = MATH_FP32, cache_enabled: bool = True, num_sessions: int = 1,
                 max_queries_per_call: int = 4096, max_histories_per_session: int = 1 << 16,
                 device: int = 0, cell: int = 0, max_queries_per_session_call: int = 0,
                 gru_path: int = GRU_AUTO):
        L = _lib.load()
        self.cfg = Config(vocab, embed, hidden, maxent_log2, maxent_order, key_mode, round_digits,
                          math, 1 if cache_enabled else 0, num_sessions, max_queries_per_call,
                          max_histories_per_session, device, cell, max_queries_per_session_call,
                          gru_path)
        self.device = torch.device("cuda", device)
        arrs = {k: np.ascontiguousarray(weights[k], dtype=np.float32) for k in _lib.WEIGHT_NAMES}
        w = Weights(**{k: arrs[k].ctypes.data_as(ctypes.c_void_p) for k in _lib.WEIGHT_NAMES})
        h = ctypes.c_void_p()
        check(L.rnnlm_create(ctypes.byref(self.cfg), ctypes.byref(w), ctypes.byref(h)),
              "rnnlm_create")
        self._h = h
        self.H = hidden
        self.N = maxent_order
        self.code_bytes = int(L.rnnlm_code_bytes(h))

    @classmethod
    def from_dims(cls, dims, weights, **kw):
        return cls(weights, vocab=dims.V, embed=dims.E, hidden=dims.H,
                   maxent_log2=dims.maxent_log2, maxent_order=dims.N, **kw)

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().rnnlm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the step ------------------------------------------------------------
    def query_batch(self, session: torch.Tensor, parent: torch.Tensor, word: torch.Tensor,
                    score: torch.Tensor | None = None, child: torch.Tensor | None = None,
                    outcome: torch.Tensor | None = None, stream=None, want_outcome: bool = True):
        n = int(word.numel())
        if score is None:
            score = torch.empty(n, dtype=torch.float32, device=self.device)
        if child is None:
            child = torch.empty(n, dtype=torch.int32, device=self.device)
        if outcome is None and want_outcome:
            outcome = torch.empty(n, dtype=torch.uint8, device=self.device)
        check(_lib.load().rnnlm_query_batch(self._h, n, _ptr(session), _ptr(parent), _ptr(word),
                                            _ptr(score), _ptr(child), _ptr(outcome),
                                            _stream(stream)), "rnnlm_query_batch")
        return score, child, outcome

    def graph(self, max_n: int, session: torch.Tensor, parent: torch.Tensor, word: torch.Tensor,
              score: torch.Tensor, child: torch.Tensor, outcome: torch.Tensor | None = None,
              n: torch.Tensor | None = None) -> "StepGraph":
        """rnnlm_graph_create: one query_batch captured on these buffers; replay
        with ``.launch()`` after rewriting their contents (and ``n``, a 1-element
        int32 device tensor holding the query count)."""
        g = ctypes.c_void_p()
        check(_lib.load().rnnlm_graph_create(self._h, int(max_n), _ptr(n), _ptr(session), _ptr(parent),
                                             _ptr(word), _ptr(score), _ptr(child), _ptr(outcome),
                                             ctypes.byref(g)), "rnnlm_graph_create")
        return StepGraph(self, g, (session, parent, word, score, child, outcome, n))

    def log_normalizer(self, session: torch.Tensor, history: torch.Tensor, out: torch.Tensor | None = None,
                       stream=None) -> torch.Tensor:
        """Exact log sum_v exp(score_v) of stored histories (rnnlm_log_normalizer)."""
        n = int(history.numel())
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=self.device)
        check(_lib.load().rnnlm_log_normalizer(self._h, n, _ptr(session), _ptr(history), _ptr(out),
                                               _stream(stream)), "rnnlm_log_normalizer")
        return out

    def results_ready(self, stream=None):
        """`stream` waits for the last query_batch's scores / handles / outcomes
        (not for its GRU state update)."""
        check(_lib.load().rnnlm_results_ready(self._h, _stream(stream)), "rnnlm_results_ready")

    def reset_session(self, session: int = ALL, stream=None):
        check(_lib.load().rnnlm_reset_session(self._h, session, _stream(stream)), "reset_session")

    def cache_stats(self, session: int = ALL) -> dict:
        st = Stats()
        _lib.load().rnnlm_cache_stats(self._h, session, ctypes.byref(st))
        return {k: int(getattr(st, k)) for k, _ in Stats._fields_ if k != "pad_"}

    # ---- inspection ------------------------------------------------------------
    def _handles(self, handles) -> torch.Tensor:
        return torch.as_tensor(np.asarray(handles, dtype=np.uint32).view(np.int32),
                               device=self.device)

    def read_states(self, session: int, handles, stream=None) -> torch.Tensor:
        h = self._handles(handles)
        out = torch.empty((h.numel(), self.H), dtype=torch.float32, device=self.device)
        check(_lib.load().rnnlm_read_states(self._h, session, h.numel(), _ptr(h), _ptr(out),
                                            _stream(stream)), "read_states")
        return out

    def read_slots(self, session: int, handles, stream=None) -> torch.Tensor:
        h = self._handles(handles)
        out = torch.empty(h.numel(), dtype=torch.int32, device=self.device)
        check(_lib.load().rnnlm_read_slots(self._h, session, h.numel(), _ptr(h), _ptr(out),
                                           _stream(stream)), "read_slots")
        return out

    def read_codes(self, session: int, handles, stream=None) -> torch.Tensor:
        h = self._handles(handles)
        out = torch.empty((h.numel(), self.code_bytes), dtype=torch.uint8, device=self.device)
        check(_lib.load().rnnlm_read_codes(self._h, session, h.numel(), _ptr(h), _ptr(out),
                                           _stream(stream)), "read_codes")
        return out

    def encode_states(self, states: torch.Tensor, stream=None) -> torch.Tensor:
        states = states.to(self.device, torch.float32).contiguous()
        n = states.shape[0]
        out = torch.empty((n, self.code_bytes), dtype=torch.uint8, device=self.device)
        check(_lib.load().rnnlm_encode_states(self._h, n, _ptr(states), _ptr(out), _stream(stream)),
              "encode_states")
        return out

    def maxent_indices(self, session, parent, word, stream=None) -> torch.Tensor:
        n = int(word.numel())
        out = torch.empty((n, self.N), dtype=torch.int64, device=self.device)
        check(_lib.load().rnnlm_maxent_indices(self._h, n, _ptr(session), _ptr(parent), _ptr(word),
                                               _ptr(out), _stream(stream)), "maxent_indices")
        return out

    # ---- timing ----------------------------------------------------------------
    def set_timing(self, level):
        check(_lib.load().rnnlm_set_timing(self._h, int(level)))

    def get_timing(self, reset: bool = True) -> dict:
        t = Timing()
        check(_lib.load().rnnlm_get_timing(self._h, ctypes.byref(t), 1 if reset else 0))
        return {k: getattr(t, k) for k, _ in Timing._fields_}

    def launch_count(self) -> int:
        return int(_lib.load().rnnlm_launch_count(self._h))

    def tf32x3_products(self) -> float:
        """Split (fp32-accurate) engines: tensor-core products per useful
        multiply-add in the mode's MMA kind (TF32X3: 3, BF16X3: 6, less the
        identically-zero ones skipped); 0 otherwise."""
        return float(_lib.load().rnnlm_tf32x3_products(self._h))


class StepGraph:
    """A captured rnnlm_query_batch (rnnlm_graph_t); keeps its buffers alive."""

    def __init__(self, eng: RNNLM, g: ctypes.c_void_p, keep):
        self.eng, self._g, self._keep = eng, g, keep

    def launch(self, stream=None):
        check(_lib.load().rnnlm_graph_launch(self._g, _stream(stream)), "rnnlm_graph_launch")

    def close(self):
        if getattr(self, "_g", None):
            _lib.load().rnnlm_graph_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def resolve_parents(ref: torch.Tensor, log: torch.Tensor, out: torch.Tensor, stream=None):
    """Workload plumbing: out[i] = ref[i] < 0 ? 0 : log[ref[i]] (int64 refs)."""
    check(_lib.load().rnnlm_resolve_parents(int(ref.numel()), _ptr(ref), _ptr(log), _ptr(out),
                                            _stream(stream)), "resolve_parents")
    return out


def as_u32(t: torch.Tensor) -> np.ndarray:
    """int32 device tensor holding u32 values -> numpy uint32."""
    return t.cpu().numpy().view(np.uint32)
