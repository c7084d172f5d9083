"""Offline level-synchronous schedule (paper_1801_09866_b200/offline.py):
host-side invariants, and on the CPU oracle the same scores as the online
(frame-by-frame) schedule when the history compression is lossless."""
import numpy as np

import oracle as O
from paper_1801_09866_b200.offline import level_schedule, levels
from synth import generate_model, generate_workload
from synth.model import ModelDims


def _wl():
    return generate_workload(3, 30, 24, 500, seed=41, dur=(2, 6))


def test_schedule_invariants():
    wl = _wl()
    lv = levels(wl.parent_ref, wl.frame_ptr)
    ref = wl.parent_ref
    has = ref >= 0
    assert np.all(lv[~has] == 0)
    assert np.all(lv[has] == lv[ref[has]] + 1)
    batches = level_schedule(wl.session, wl.parent_ref, wl.frame_ptr, max_batch=40)
    seen = np.full(wl.n_total, -1)
    for b, ix in enumerate(batches):
        assert len(ix) <= 40
        seen[ix] = b
        s = wl.session[ix]
        assert np.all(np.diff(s.astype(np.int64)) >= 0)                      # sorted by session
        for sv in np.unique(s):
            assert np.all(np.diff(ix[s == sv]) > 0)                         # stream order inside
    assert np.all(seen >= 0)
    p = ref >= 0
    assert np.all(seen[ref[p]] < seen[p])                                   # parents in earlier calls
    # one level per word boundary of the deepest path: fewer levels than frames
    assert lv.max() + 1 < wl.frames
    assert len(level_schedule(wl.session, wl.parent_ref, wl.frame_ptr, 1 << 30)) == lv.max() + 1


def test_oracle_offline_equals_online_lossless():
    """Mode off: a score depends only on (parent state, word) and a state only
    on (parent state, word), so running the same stream level by level must
    give every query bitwise the same score as running it frame by frame."""
    d = ModelDims(V=500, E=16, H=16, maxent_log2=12, N=3)
    m = generate_model(d, seed=5, scale=1.0)
    wl = _wl()
    cap = wl.n_total + 2
    cfg = O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_OFF, 0, 1, wl.S, cap)
    on = O.Oracle(cfg, m)
    child_on = np.zeros(wl.n_total, np.uint32)
    score_on = np.zeros(wl.n_total, np.float32)
    for t in range(wl.frames):
        sl = wl.frame_slice(t)
        par = O.resolve_parents(wl.parent_ref[sl], child_on)
        sc, ch, _ = on.query_frame(wl.session[sl], par, wl.word[sl])
        score_on[sl], child_on[sl] = sc, ch
    off = O.Oracle(cfg, m)
    child_off = np.zeros(wl.n_total, np.uint32)
    score_off = np.zeros(wl.n_total, np.float32)
    for ix in level_schedule(wl.session, wl.parent_ref, wl.frame_ptr, max_batch=50):
        par = O.resolve_parents(wl.parent_ref[ix], child_off)
        sc, ch, _ = off.query_frame(wl.session[ix], par, wl.word[ix])
        score_off[ix], child_off[ix] = sc, ch
    assert np.array_equal(score_on.view(np.uint32), score_off.view(np.uint32))
    # the children carry the same states (handle numbering differs between schedules)
    for s in range(wl.S):
        msk = wl.session == s
        a = on.read_states(s, child_on[msk])
        b = off.read_states(s, child_off[msk])
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
