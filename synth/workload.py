"""Seeded LibriSpeech-shaped LM-query streams (stand-in for a WFST decoder).

The paper's queries come from a live CPU-GPU WFST decoder that emits word
hypotheses at word boundaries during frame-synchronous Viterbi search
(P:45-46); no trace format exists, so this generator is an invention
(SURVEY 8(d)).  What it reproduces:

* frame structure: one batch of queries per 10 ms decoder frame;
  a 4-s utterance is 400 frames;
* beam structure: P hypothesis paths per utterance; a path at a word
  boundary emits K candidate next words (Zipf(1.0) over word ids 1..V-1)
  against its current history, then advances to the child of one of them
  (the transcript word with probability 1-eps, else a substitution);
* repeated queries: the same (history, word) pair is re-emitted in later
  frames (word-end-time ambiguity), which is what the paper's LM-query cache
  removes (~89% hits).  Re-emissions fill each frame up to exactly
  B_s queries per session, so the hit ratio is ~ 1 - P*K/(mean_dur*B_s);
* shared recent pasts: every path starts with ``private`` words of its own
  (hypotheses that differ in earlier context), then all paths of an
  utterance follow the same transcript with independent substitutions, so
  histories that differ in an older word share their recent words (what
  lossy history keys merge).

Parents are expressed as *references to earlier queries* (``parent_ref`` =
flat index of the query whose returned child handle is the parent history,
-1 = the utterance root).  The consumer (bench / tests) maps references to
handles with the handles the engine under test returned, so this module
never simulates any part of the method.  Parents always come from earlier
frames (SURVEY 8(c) reading 17).
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class Workload:
    S: int                 # sessions (utterance streams)
    B_s: int               # queries per session per frame
    frames: int
    V: int
    session: np.ndarray    # uint32 [frames*S*B_s], session-major inside a frame
    parent_ref: np.ndarray  # int64, -1 = root history
    word: np.ndarray       # uint32
    new_per_session: np.ndarray  # int64 [S]: number of first emissions (>= distinct pairs)

    @property
    def n_per_frame(self) -> int:
        return self.S * self.B_s

    @property
    def n_total(self) -> int:
        return self.frames * self.n_per_frame

    def frame_slice(self, t: int) -> slice:
        n = self.n_per_frame
        return slice(t * n, (t + 1) * n)

    def max_histories_hint(self) -> int:
        """Upper bound on history handles any session can need (+root)."""
        return int(self.new_per_session.max()) + 2

    def select_sessions(self, lo: int, hi: int) -> "Workload":
        """Sessions [lo, hi) as their own workload (references re-based)."""
        S2 = hi - lo
        sel = []
        remap = np.full(self.n_total, -1, dtype=np.int64)
        for t in range(self.frames):
            base = t * self.n_per_frame
            idx = np.arange(base + lo * self.B_s, base + hi * self.B_s)
            remap[idx] = t * S2 * self.B_s + np.arange(S2 * self.B_s)
            sel.append(idx)
        sel = np.concatenate(sel) if sel else np.zeros(0, dtype=np.int64)
        pr = self.parent_ref[sel]
        pr2 = np.where(pr >= 0, remap[np.maximum(pr, 0)], -1)
        return Workload(S=S2, B_s=self.B_s, frames=self.frames, V=self.V,
                        session=(self.session[sel] - lo).astype(np.uint32),
                        parent_ref=pr2.astype(np.int64), word=self.word[sel].copy(),
                        new_per_session=self.new_per_session[lo:hi].copy())


def _zipf_cdf(V: int, s: float) -> np.ndarray:
    ranks = np.arange(1, V, dtype=np.float64)
    p = ranks ** (-s)
    c = np.cumsum(p)
    return c / c[-1]


def generate_workload(S: int, frames: int, B_s: int, V: int, seed: int = 7,
                      K: int = 8, dur: tuple = (10, 40), eps: float = 0.3,
                      window: int = 12, zipf_s: float = 1.0,
                      qhit_target: float = 0.87, private: int = 2) -> Workload:
    """Session s draws from its own generator seeded ``seed + s``."""
    assert V >= 2 and B_s >= 1 and S >= 1 and frames >= 0
    cdf = _zipf_cdf(V, zipf_s)
    mean_dur = 0.5 * (dur[0] + dur[1])
    P = max(1, int(round(B_s * (1.0 - qhit_target) * mean_dur / K)))
    n_frame = S * B_s
    session = np.repeat(np.arange(S, dtype=np.uint32), B_s)
    session = np.tile(session, frames)
    parent_ref = np.empty(frames * n_frame, dtype=np.int64)
    word = np.empty(frames * n_frame, dtype=np.uint32)
    new_count = np.zeros(S, dtype=np.int64)

    def zipf(rng, n):
        return (np.searchsorted(cdf, rng.random(n), side="right") + 1).astype(np.int64).clip(1, V - 1)

    for s in range(S):
        rng = np.random.default_rng(seed + s)
        transcript = zipf(rng, frames // max(1, dur[0]) + 8)
        # each path first emits `private` words of its own (hypotheses that
        # differ in their earlier context), then follows the shared transcript
        own = zipf(rng, P * private).reshape(P, private) if private else None
        path_ref = np.full(P, -1, dtype=np.int64)
        path_pos = np.full(P, -private, dtype=np.int64)
        next_b = rng.integers(0, dur[1], size=P)
        recent = []  # list of (parent_refs, words) of first emissions, last `window` frames
        for t in range(frames):
            base = t * n_frame + s * B_s
            bpaths = np.nonzero(next_b == t)[0]
            max_paths = B_s // K if B_s >= K else 0
            if len(bpaths) > max_paths:      # frame full: postpone the rest
                next_b[bpaths[max_paths:]] = t + 1
                bpaths = bpaths[:max_paths]
            nb = len(bpaths)
            if nb:
                cand = zipf(rng, nb * K).reshape(nb, K)
                pos = path_pos[bpaths]
                cand[:, 0] = np.where(
                    pos < 0, own[bpaths, np.clip(pos + private, 0, private - 1)] if private else 0,
                    transcript[np.clip(pos, 0, len(transcript) - 1)])
                new_par = np.repeat(path_ref[bpaths], K)
                new_w = cand.reshape(-1)
            else:
                new_par = np.zeros(0, dtype=np.int64)
                new_w = np.zeros(0, dtype=np.int64)
            m = len(new_w)
            pool_p = [r[0] for r in recent] + [new_par]
            pool_w = [r[1] for r in recent] + [new_w]
            pool_p = np.concatenate(pool_p)
            pool_w = np.concatenate(pool_w)
            n_rep = B_s - m
            if len(pool_p) == 0:             # nothing emitted yet: root queries
                pool_p = np.full(1, -1, dtype=np.int64)
                pool_w = zipf(rng, 1)
            ri = rng.integers(0, len(pool_p), size=n_rep)
            fp = np.concatenate([new_par, pool_p[ri]])
            fw = np.concatenate([new_w, pool_w[ri]])
            perm = rng.permutation(B_s)      # position j holds query perm[j]
            parent_ref[base:base + B_s] = fp[perm]
            word[base:base + B_s] = fw[perm]
            if nb:
                pos_of = np.empty(B_s, dtype=np.int64)
                pos_of[perm] = np.arange(B_s)
                choice = np.where(rng.random(nb) < eps, rng.integers(1, K, size=nb), 0)
                chosen_new_idx = np.arange(nb) * K + choice
                path_ref[bpaths] = base + pos_of[chosen_new_idx]
                path_pos[bpaths] += 1
                next_b[bpaths] = t + rng.integers(dur[0], dur[1] + 1, size=nb)
            new_count[s] += m
            recent.append((new_par, new_w))
            if len(recent) > window:
                recent.pop(0)
    return Workload(S=S, B_s=B_s, frames=frames, V=V, session=session,
                    parent_ref=parent_ref, word=word, new_per_session=new_count + 1)

