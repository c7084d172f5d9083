"""Offline (2-pass) rescoring schedule -- SURVEY 8(f)-4.

The paper rescores ONLINE: one call per decoder frame, because the next
frame's hypotheses are not known yet; a 2-pass decoder "could not
be applied before the end of the utterance was reached".  When the
whole utterance's query stream IS known (lattice rescoring after the first
pass), a query depends only on its parent history, so queries can be grouped
by dependency level instead of by frame:

    level(q) = 0                       if q's parent is the utterance root,
             = level(parent query) + 1 otherwise,

and every level is one batch (split at ``max_batch``; inside a batch the
queries are ordered by session, then stream order, as rnnlm_query_batch
requires).  Parents always sit in earlier batches (reading 17), the
number of calls drops from #frames to #levels, and each call carries a much
larger GRU block -- the per-frame latency bound of the online path goes away.
Host-side scheduling only: every step of the path still runs in the library's
kernels; the gather / scatter of the batches' inputs and results are plain
device tensor indexing (plumbing).

Semantics: with lossless keys (off) every query gets bitwise its online score
and state.  With lossy keys (sign / round) the first occupant of a
hidden-cache key, and so which histories share a state, follows the LEVEL
order, and handles are numbered in that order: results can differ from the
online (frame-order) run; they equal the oracle replaying the same schedule
(tests: test_offline_level_batches_vs_oracle, every key mode).
"""
from __future__ import annotations

import numpy as np
import torch

from . import engine as _engine


def levels(parent_ref: np.ndarray, frame_ptr: np.ndarray) -> np.ndarray:
    """Dependency level of every query (int32); parents reference earlier frames
    (frame t = queries [frame_ptr[t], frame_ptr[t+1]))."""
    n = parent_ref.shape[0]
    lv = np.zeros(n, dtype=np.int32)
    for lo, hi in zip(frame_ptr[:-1], frame_ptr[1:]):
        ref = parent_ref[lo:hi]
        lv[lo:hi] = np.where(ref < 0, 0, lv[np.maximum(ref, 0)] + 1)
    return lv


def level_schedule(session: np.ndarray, parent_ref: np.ndarray, frame_ptr: np.ndarray,
                   max_batch: int) -> list:
    """Batches (int64 index arrays) in execution order: by level, then session,
    then stream order; a level larger than ``max_batch`` is split."""
    lv = levels(parent_ref, frame_ptr)
    idx = np.arange(lv.shape[0], dtype=np.int64)
    order = np.lexsort((idx, session.astype(np.int64), lv.astype(np.int64)))
    lvs = lv[order]
    cuts = np.flatnonzero(np.diff(lvs)) + 1
    out = []
    for part in np.split(order, cuts):
        for lo in range(0, part.shape[0], max_batch):
            out.append(part[lo:lo + max_batch])
    return out


class OfflineRunner:
    """Runs a workload's whole query stream through an engine level by level.
    Results land at the queries' stream positions (``score``, ``child``)."""

    def __init__(self, eng: "_engine.RNNLM", wl, max_batch: int, device=None):
        self.eng = eng
        self.device = device or eng.device
        self.batches = level_schedule(wl.session, wl.parent_ref, wl.frame_ptr, max_batch)
        dev = self.device
        self.d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
        self.d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
        self.d_ref = torch.as_tensor(wl.parent_ref, device=dev)
        self.d_idx = [torch.as_tensor(b, device=dev) for b in self.batches]
        self.score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
        self.child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
        m = max((b.shape[0] for b in self.batches), default=0)
        self._par = torch.zeros(m, dtype=torch.int32, device=dev)
        self._sc = torch.zeros(m, dtype=torch.float32, device=dev)
        self._ch = torch.zeros(m, dtype=torch.int32, device=dev)

    def run(self):
        for ix in self.d_idx:
            k = ix.shape[0]
            par, sc, ch = self._par[:k], self._sc[:k], self._ch[:k]
            _engine.resolve_parents(self.d_ref[ix], self.child, par)
            self.eng.query_batch(self.d_sess[ix], par, self.d_word[ix], score=sc, child=ch, want_outcome=False)
            self.score[ix] = sc
            self.child[ix] = ch
        return self.score, self.child
