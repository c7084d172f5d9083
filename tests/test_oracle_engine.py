"""Pins of the oracle's cache/bookkeeping semantics.

Expected values are hand-enumerated frames, counting laws, brute-force
enumeration of keys, and the equivalence the paper's method guarantees when
compression is lossless (mode off == no cache, BASELINE.json north_star).
"""
import itertools

import numpy as np
import pytest

import oracle as O
from synth import generate_workload
from synth.model import ModelDims, generate_model

QHIT, SHIT, MISS, INV = O.QHIT, O.SHIT, O.MISS, O.INVALID


def engine(dims, model, mode=O.KEY_OFF, k=0, cache=1, S=1, cap=1 << 16):
    cfg = O.make_config(dims.V, dims.E, dims.H, dims.maxent_log2, dims.N, mode, k, cache, S, cap)
    return O.Oracle(cfg, model)


@pytest.fixture(scope="module")
def small():
    d = ModelDims(V=16, E=8, H=8, maxent_log2=8, N=3)
    return d, generate_model(d, seed=1234, scale=0.5)


def test_hand_frame_handles_and_outcomes(small):
    d, m = small
    e = engine(d, m)
    # frame 1 (all parents = root 0): (0,5) (0,6) (0,5) (0,7)
    sc, ch, oc = e.query_frame([0] * 4, [0, 0, 0, 0], [5, 6, 5, 7])
    assert oc.tolist() == [MISS, MISS, QHIT, MISS]        # dup -> query-cache hit
    assert ch.tolist() == [1, 2, 1, 3]                    # dense, non-QHIT only (reading 20)
    assert sc[0] == sc[2]
    assert e.stats() == dict(total_queries=4, query_hits=1, hidden_lookups=3, hidden_hits=0,
                             gru_computations=3, sticky_error=0)
    # frame 2: parent 4 does not exist yet; word 99 >= V
    sc, ch, oc = e.query_frame([0] * 6, [1, 2, 3, 0, 4, 1], [9, 9, 9, 5, 1, 99])
    assert oc.tolist() == [MISS, MISS, MISS, QHIT, INV, INV]
    assert ch.tolist() == [4, 5, 6, 1, 0xFFFFFFFF, 0xFFFFFFFF]
    assert np.isnan(sc[4]) and np.isnan(sc[5])
    st = e.stats()
    assert st["total_queries"] == 8 and st["query_hits"] == 2 and st["gru_computations"] == 6
    assert st["sticky_error"] == 5                        # E_HISTORY latched first
    # parent created earlier in the SAME frame is rejected (reading 17)
    _, ch2, oc2 = e.query_frame([0, 0], [6, 7], [1, 1])
    assert oc2.tolist() == [MISS, INV]
    # contexts: handle 1 = [0,5]; handle 4 = (ctx of 1) o 9 -> last 2 = [5,9]
    assert e.read_ctx(0, [0, 1, 4]) == [[0], [0, 5], [5, 9]]


def test_child_state_is_gru_of_parent(small):
    d, m = small
    e = engine(d, m)
    e.query_frame([0], [0], [3])
    e.query_frame([0], [1], [4])
    cfg = O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N)
    h1 = O.gru(cfg, m, m["emb"][3], np.zeros(d.H, np.float32))
    h2 = O.gru(cfg, m, m["emb"][4], h1)
    st = e.read_states(0, [0, 1, 2])
    assert np.array_equal(st[0], np.zeros(d.H)) and np.array_equal(st[1], h1)
    assert np.array_equal(st[2], h2)
    # score conditions on the PARENT (reading 2): query (1, 4) scored with h1, ctx [0,3]
    e.query_frame([0], [1], [7])
    sc, _, oc = e.query_frame([0], [1], [7])
    assert oc[0] == QHIT and sc[0] == np.float32(O.score(cfg, m, h1, [0, 3], 7))


def _chain_workload(frames_half, width, V):
    """All (parent, word) pairs distinct in the first half; second half replays it."""
    par, wrd = [], []
    for t in range(frames_half):
        for j in range(width):
            par.append(-1 if t == 0 else (t - 1) * width + j)
            wrd.append((t * width + j) % (V - 1) + 1)
    par = np.array(par, np.int64)
    wrd = np.array(wrd, np.uint32)
    return np.concatenate([par, par]), np.concatenate([wrd, wrd])


def test_repetition_hit_ratio_S566(small):
    d, m = small
    e = engine(d, m)
    width, half = 6, 5
    par_ref, wrd = _chain_workload(half, width, d.V)
    child = np.zeros(len(wrd), np.uint32)
    for t in range(2 * half):
        sl = slice(t * width, (t + 1) * width)
        _, ch, _ = e.query_frame(np.zeros(width), O.resolve_parents(par_ref[sl], child), wrd[sl])
        child[sl] = ch
        if t == half - 1:
            first = e.stats()
    st = e.stats()
    assert first["query_hits"] == 0
    assert st["query_hits"] / st["total_queries"] == 0.5
    assert (st["query_hits"] - first["query_hits"]) / (st["total_queries"] - first["total_queries"]) == 1.0


@pytest.mark.parametrize("mode,k", [(O.KEY_OFF, 0), (O.KEY_SIGN, 0), (O.KEY_ROUND, 1),
                                    (O.KEY_ROUND, 2), (O.KEY_ROUND, 3)])
def test_stats_identities_and_coarsening(small, mode, k):
    d, m = small
    wl = generate_workload(2, 30, 24, d.V, seed=3)
    res = {}
    for mm, kk in ((O.KEY_OFF, 0), (mode, k)):
        e = engine(d, m, mm, kk, S=2)
        O.run_workload(e, wl)
        st = e.stats()
        # S:255
        assert st["hidden_lookups"] + st["query_hits"] == st["total_queries"] == wl.n_total
        assert st["gru_computations"] + st["hidden_hits"] == st["hidden_lookups"]
        res[(mm, kk)] = st
    # coarsening: a key that is a function of the exact key can only merge
    assert res[(mode, k)]["gru_computations"] <= res[(O.KEY_OFF, 0)]["gru_computations"]
    # the LM-query cache is exact: same hits whatever the history key
    assert res[(mode, k)]["query_hits"] == res[(O.KEY_OFF, 0)]["query_hits"]


def test_mode_off_equals_no_cache_bitwise(small):
    """Cache-hit equivalence (BASELINE north_star)."""
    d, m = small
    wl = generate_workload(2, 25, 20, d.V, seed=5)
    e_on = engine(d, m, O.KEY_OFF, 0, cache=1, S=2)
    e_off = engine(d, m, O.KEY_OFF, 0, cache=0, S=2)
    s1, c1, o1 = O.run_workload(e_on, wl)
    s2, c2, o2 = O.run_workload(e_off, wl)
    assert np.array_equal(s1.view(np.uint32), s2.view(np.uint32))
    assert set(o2.tolist()) == {MISS}
    for s in range(2):
        idx = np.nonzero(wl.session == s)[0]
        a = e_on.read_states(s, c1[idx])
        b = e_off.read_states(s, c2[idx])
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    st = e_off.stats()
    assert st["query_hits"] == 0 and st["gru_computations"] == wl.n_total


def test_sign_pigeonhole_and_bruteforce_key_count():
    """H=8, V=4: unique GRU computations = #distinct (word, sign code) keys <= 2^8*4."""
    d = ModelDims(V=4, E=4, H=8, maxent_log2=6, N=2)
    m = generate_model(d, seed=9, scale=1.0, bf16_grid=False)
    e = engine(d, m, O.KEY_SIGN)
    rng = np.random.default_rng(0)
    handles = [0]
    keys = set()
    for t in range(40):
        par = rng.choice(handles, size=64)
        wrd = rng.integers(0, 4, size=64)
        # brute force: the key of every query that will reach the hidden cache
        states = e.read_states(0, par)
        before = e.stats()
        _, ch, oc = e.query_frame(np.zeros(64), par, wrd)
        for i in range(64):
            if oc[i] != QHIT:
                keys.add((int(wrd[i]), O.compress(states[i], O.KEY_SIGN).tobytes()))
        handles.extend(int(c) for c in set(ch.tolist()) if c not in handles)
    st = e.stats()
    assert st["gru_computations"] == len(keys)
    assert st["gru_computations"] <= 2 ** 8 * 4


def test_sign_merge_construction_S284():
    """States differing by |delta| < 1e-3, every |h_i| > 1e-3: hit under sign, miss under off."""
    d = ModelDims(V=512, E=4, H=16, maxent_log2=6, N=2)
    m = generate_model(d, seed=2)
    rng = np.random.default_rng(3)
    n = 200
    for mode, expect in ((O.KEY_SIGN, SHIT), (O.KEY_OFF, MISS)):
        e = engine(d, m, mode)
        _, ch, _ = e.query_frame(np.zeros(2 * n), np.zeros(2 * n), np.arange(1, 2 * n + 1))
        for i in range(n):
            mag = rng.uniform(2e-3, 0.9, d.H) * rng.choice([-1, 1], d.H)
            delta = rng.uniform(-9.9e-4, 9.9e-4, d.H)
            e.overwrite_state(0, int(ch[2 * i]), mag.astype(np.float32))
            e.overwrite_state(0, int(ch[2 * i + 1]), (mag + delta).astype(np.float32))
        _, ch2, oc2 = e.query_frame(np.zeros(2 * n), ch, np.full(2 * n, 3))
        assert set(oc2[0::2].tolist()) == {MISS}
        assert set(oc2[1::2].tolist()) == {expect}
        if expect == SHIT:
            s1 = e.read_slots(0, ch2[0::2])
            s2 = e.read_slots(0, ch2[1::2])
            assert np.array_equal(s1, s2)                  # first occupant's state (reading 8)


def test_tiny_vocab_bruteforce_all_sequences():
    """V=4: every word sequence of length <= 3, frame by frame, vs direct chaining."""
    d = ModelDims(V=4, E=3, H=4, maxent_log2=5, N=3)
    m = generate_model(d, seed=8, scale=0.8, bf16_grid=False)
    cfg = O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N)
    for cache in (1, 0):
        e = engine(d, m, O.KEY_OFF, cache=cache)
        frontier = {(): 0}                    # word sequence -> handle
        for depth in range(3):
            seqs = [s + (w,) for s in frontier for w in range(4)]
            par = [frontier[s[:-1]] for s in seqs]
            sc, ch, oc = e.query_frame(np.zeros(len(seqs)), par, [s[-1] for s in seqs])
            assert INV not in oc.tolist()
            for i, s in enumerate(seqs):
                h = np.zeros(d.H, np.float32)
                ctx = [0]
                for w in s[:-1]:
                    h = O.gru(cfg, m, m["emb"][w], h)
                    ctx = (ctx + [w])[-(d.N - 1):]
                assert sc[i] == np.float32(O.score(cfg, m, h, ctx, s[-1]))
                hc = O.gru(cfg, m, m["emb"][s[-1]], h)
                assert np.array_equal(e.read_states(0, [ch[i]])[0], hc)
            frontier = {s: int(ch[i]) for i, s in enumerate(seqs)}


def test_capacity_overflow_sets_sticky(small):
    d, m = small
    e = engine(d, m, cap=4)
    _, ch, oc = e.query_frame(np.zeros(5), np.zeros(5), [1, 2, 3, 4, 1])
    assert oc.tolist() == [MISS, MISS, MISS, INV, QHIT]
    assert e.stats()["sticky_error"] == 6


def test_reset_session_clears(small):
    d, m = small
    e = engine(d, m, S=2)
    e.query_frame([0, 1], [0, 0], [1, 1])
    e.reset_session(0)
    assert e.num_handles(0) == (1, 1) and e.num_handles(1) == (2, 2)
    assert e.stats(0)["total_queries"] == 0 and e.stats(1)["total_queries"] == 1


def test_staggered_and_selected_workloads_are_well_formed():
    """Workload plumbing used by bench.py / the GPU tests: every frame of a
    staggered or session-selected stream is sorted by session (reading 24),
    parents come from earlier frames of the same session (reading 17), and a
    stream keeps its own query sequence."""
    wl = generate_workload(3, 20, 16, 1000, seed=7)
    st = wl.staggered([0, 5, 10])
    for w in (st, st.select_sessions(1, 3), wl.select_sessions(0, 2)):
        f = w.frame_index()
        for t in range(w.frames):
            s = w.session[w.frame_slice(t)].astype(np.int64)
            assert np.all(np.diff(s) >= 0)
        m = w.parent_ref >= 0
        assert np.all(f[w.parent_ref[m]] < f[m])
        assert np.all(w.session[w.parent_ref[m]] == w.session[m])
    a, b = wl.select_sessions(1, 2), st.select_sessions(1, 2)
    assert np.array_equal(a.word[:b.n_total], b.word) and np.array_equal(a.parent_ref[:b.n_total], b.parent_ref)


def test_threaded_frames_equal_single_thread():
    """The oracle evaluates a frame's scores and GRUs after its (sequential)
    decisions, optionally on several host threads (bench.py's cpu_baseline);
    the arithmetic of each item is unchanged, so results are bitwise those of
    one thread."""
    d = ModelDims(V=500, E=32, H=32, maxent_log2=12, N=3)
    m = generate_model(d, seed=3)
    wl = generate_workload(2, 30, 64, d.V, seed=5, dur=(2, 6), eps=0.1)
    outs = []
    old = O.threads()
    try:
        for th in (1, 4):
            O.threads(th)
            orc = engine(d, m, O.KEY_SIGN, S=2, cap=wl.max_histories_hint())
            child = np.zeros(wl.n_total, np.uint32)
            score = np.zeros(wl.n_total, np.float32)
            for t in range(wl.frames):
                sl = wl.frame_slice(t)
                par = O.resolve_parents(wl.parent_ref[sl], child)
                sc, ch, _ = orc.query_frame(wl.session[sl], par, wl.word[sl])
                score[sl], child[sl] = sc, ch
            outs.append((score, orc.read_states(0, np.arange(orc.num_handles(0)[0], dtype=np.uint32)), orc.stats()))
    finally:
        O.threads(old)
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1].view(np.uint32), outs[1][1].view(np.uint32))
    assert outs[0][2] == outs[1][2]
