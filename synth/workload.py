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
    B_s: int               # queries per session per frame (at most)
    frames: int
    V: int
    session: np.ndarray    # uint32, session-major inside a frame
    parent_ref: np.ndarray  # int64, -1 = root history
    word: np.ndarray       # uint32
    new_per_session: np.ndarray  # int64 [S]: number of first emissions (>= distinct pairs)
    frame_ptr: np.ndarray = None  # int64 [frames+1]: frame t = queries [ptr[t], ptr[t+1]); None = S*B_s each

    def __post_init__(self):
        if self.frame_ptr is None:
            self.frame_ptr = np.arange(self.frames + 1, dtype=np.int64) * (self.S * self.B_s)

    @property
    def n_per_frame(self) -> int:
        """The largest frame (sizes the engine's max_queries_per_call)."""
        return int(np.max(np.diff(self.frame_ptr))) if self.frames else 0

    @property
    def n_total(self) -> int:
        return int(self.frame_ptr[-1])

    def frame_slice(self, t: int) -> slice:
        return slice(int(self.frame_ptr[t]), int(self.frame_ptr[t + 1]))

    def max_histories_hint(self) -> int:
        """Upper bound on history handles any session can need (+root)."""
        return int(self.new_per_session.max()) + 2

    def _select(self, keep: np.ndarray, frame_of: np.ndarray, frames: int, session: np.ndarray,
                S: int, new_per_session: np.ndarray) -> "Workload":
        """Queries with keep[i], placed in frame frame_of[i] (inside a frame:
        session-major, stream order within a session -- the order
        rnnlm_query_batch requires), references re-based; a kept query's parent
        must be kept."""
        idx = np.nonzero(keep)[0]
        order = idx[np.lexsort((idx, session[idx], frame_of[idx]))]
        remap = np.full(self.n_total, -1, dtype=np.int64)
        remap[order] = np.arange(len(order))
        pr = self.parent_ref[order]
        pr2 = np.where(pr >= 0, remap[np.maximum(pr, 0)], -1)
        assert not np.any((pr >= 0) & (pr2 < 0)), "a kept query's parent was dropped"
        ptr = np.searchsorted(frame_of[order], np.arange(frames + 1), side="left").astype(np.int64)
        return Workload(S=S, B_s=self.B_s, frames=frames, V=self.V,
                        session=session[order].astype(np.uint32), parent_ref=pr2.astype(np.int64),
                        word=self.word[order].copy(), new_per_session=new_per_session, frame_ptr=ptr)

    def frame_index(self) -> np.ndarray:
        """Frame of every query."""
        return np.repeat(np.arange(self.frames, dtype=np.int64), np.diff(self.frame_ptr))

    def select_sessions(self, lo: int, hi: int) -> "Workload":
        """Sessions [lo, hi) as their own workload (references re-based)."""
        keep = (self.session >= lo) & (self.session < hi)
        return self._select(keep, self.frame_index(), self.frames,
                            (self.session.astype(np.int64) - lo), hi - lo,
                            self.new_per_session[lo:hi].copy())

    def staggered(self, starts) -> "Workload":
        """Concurrent streams that are not in step (BASELINE configs[4]): session s
        joins at global frame starts[s] with its utterance's frame 0, so at global
        frame t it is at utterance frame t - starts[s]; every frame of the result
        keeps the S*B_s layout once all sessions have joined.  Same number of
        global frames; session s keeps its first frames - starts[s] frames."""
        starts = np.asarray(starts, dtype=np.int64)
        assert len(starts) == self.S and np.all(starts >= 0) and np.all(starts < max(1, self.frames))
        f = self.frame_index()
        g = f + starts[self.session.astype(np.int64)]
        keep = g < self.frames
        return self._select(keep, g, self.frames, self.session, self.S, self.new_per_session.copy())


def _zipf_cdf(V: int, s: float) -> np.ndarray:
    ranks = np.arange(1, V, dtype=np.float64)
    p = ranks ** (-s)
    c = np.cumsum(p)
    return c / c[-1]


def generate_workload(S: int, frames: int, B_s: int, V: int, seed: int = 7,
                      K: int = 8, dur: tuple = (10, 40), eps: float = 0.28,
                      window: int = 12, zipf_s: float = 1.0,
                      qhit_target: float = 0.88, n_alt: int = 2,
                      beam_scale: float = 1.8) -> Workload:
    """Session s draws from its own generator seeded ``seed + s``.

    Lattice-shaped beam: per session a transcript of
    Zipf words; transcript position j has ``n_alt`` confusable alternatives
    and a candidate set C_j of K words (the transcript word, its
    alternatives, K-1-n_alt other Zipf words) that is the SAME for every path
    reaching position j -- the acoustic evidence proposes the words, not the
    LM history.  P beam paths walk the positions at their own word-boundary
    times (``dur`` frames per word); at a boundary a path emits (history, w)
    for every w in C_j and then takes the transcript word with probability
    1 - eps, else one of the alternatives.  Paths therefore differ in a few
    confusion positions and agree elsewhere: histories that differ only in
    an older word share their recent words, which is what lossy history keys
    merge (Table 1).  ``beam_scale`` sets P relative to the
    number of first emissions a ``qhit_target`` query-cache hit ratio needs
    (paths with identical histories emit identical queries, so the measured
    ratio is higher; eps = 0.28, beam_scale = 1.8 give ~0.88 and ~15 % sign
    redundancy at H = 256).
    """
    assert V >= 2 and B_s >= 1 and S >= 1 and frames >= 0
    assert K >= 1 + n_alt
    cdf = _zipf_cdf(V, zipf_s)
    mean_dur = 0.5 * (dur[0] + dur[1])
    P = max(1, int(round(beam_scale * B_s * (1.0 - qhit_target) * mean_dur / K)))
    n_frame = S * B_s
    session = np.repeat(np.arange(S, dtype=np.uint32), B_s)
    session = np.tile(session, frames)
    parent_ref = np.empty(frames * n_frame, dtype=np.int64)
    word = np.empty(frames * n_frame, dtype=np.uint32)
    new_count = np.zeros(S, dtype=np.int64)
    L = frames // max(1, dur[0]) + 8                     # transcript positions a path can reach

    def zipf(rng, n):
        return (np.searchsorted(cdf, rng.random(n), side="right") + 1).astype(np.int64).clip(1, V - 1)

    for s in range(S):
        rng = np.random.default_rng(seed + s)
        cands = zipf(rng, L * K).reshape(L, K)           # column 0: transcript, 1..n_alt: confusions
        path_ref = np.full(P, -1, dtype=np.int64)        # -1 = the utterance root
        path_pos = np.zeros(P, dtype=np.int64)
        next_b = rng.integers(0, dur[1], size=P)
        recent = []  # (parent_refs, words) of first emissions, last `window` frames
        for t in range(frames):
            base = t * n_frame + s * B_s
            bpaths = np.nonzero(next_b == t)[0]
            max_paths = B_s // K if B_s >= K else 0
            if len(bpaths) > max_paths:      # frame full: postpone the rest
                next_b[bpaths[max_paths:]] = t + 1
                bpaths = bpaths[:max_paths]
            nb = len(bpaths)
            new_par = np.repeat(path_ref[bpaths], K)
            new_w = cands[np.minimum(path_pos[bpaths], L - 1)].reshape(-1)
            m = len(new_w)
            pool_p = np.concatenate([r[0] for r in recent] + [new_par])
            pool_w = np.concatenate([r[1] for r in recent] + [new_w])
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
                choice = np.where(rng.random(nb) < eps, rng.integers(1, 1 + n_alt, size=nb), 0)
                path_ref[bpaths] = base + pos_of[np.arange(nb) * K + choice]
                path_pos[bpaths] += 1
                next_b[bpaths] = t + rng.integers(dur[0], dur[1] + 1, size=nb)
            new_count[s] += m
            recent.append((new_par, new_w))
            if len(recent) > window:
                recent.pop(0)
    return Workload(S=S, B_s=B_s, frames=frames, V=V, session=session,
                    parent_ref=parent_ref, word=word, new_per_session=new_count + 1)
