"""GPU parity: the CUDA path through the C ABI vs the CPU oracle.

Bar (BASELINE.json north_star): bit-exact keys, MaxEnt indices, outcomes,
handles, slots, stats; scores and states within 1e-5 (FP32 path) / 1e-3
(BF16 and TF32 tensor-core paths).  Inputs: seeded synth/ generators with the shapes of
the BASELINE.json configs.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1801_09866_b200 import (KEY_OFF, KEY_ROUND, KEY_SIGN, MATH_BF16, MATH_BF16X3, MATH_FP32, MATH_TF32, MATH_TF32X3, RNNLM,
                                   INVALID, MISS, QHIT, SHIT, GRU_GEMV, GRU_TILES)
from synth import generate_model, generate_workload, model_dims
from synth.model import ModelDims
from tests.parity_util import _dev, replay_compare

pytestmark = pytest.mark.gpu

TOL = {MATH_FP32: 1e-5, MATH_BF16: 1e-3, MATH_TF32: 1e-3,    # 1e-3 for bf16/tf32
       MATH_TF32X3: 1e-5, MATH_BF16X3: 1e-5}                   # fp32-accurate tensor-core modes: the FP32 bar
_models = {}


def model(name_or_dims, seed=1234, scale=None):
    key = (name_or_dims, seed, scale)
    if key not in _models:
        d = model_dims(name_or_dims) if isinstance(name_or_dims, str) else name_or_dims
        _models[key] = (d, generate_model(d, seed=seed, scale=scale))
    return _models[key]


def lattice(S, F, B, V, seed):
    """A stream with many GRU rows early on: short words (2-6 frames) and
    substitution rate 0.1, so 8-40 frames already hold several words per path."""
    return generate_workload(S, F, B, V, seed=seed, dur=(2, 6), eps=0.1)


def pair(d, m, wl, mode=KEY_OFF, k=0, math=MATH_FP32, cache=True, B=None, cap=None, cell=0, path=GRU_TILES):
    """An engine (GRU kernels: ``path``; the tile kernels unless a test asks
    for the small-frame GEMV kernels) and an oracle over the same model."""
    cap = cap or (wl.max_histories_hint() if cache else wl.n_total // wl.S + 2)
    B = B or wl.n_per_frame
    eng = RNNLM.from_dims(d, m, key_mode=mode, round_digits=k, math=math, cache_enabled=cache,
                          num_sessions=wl.S, max_queries_per_call=B, max_histories_per_session=cap, cell=cell,
                          gru_path=path)
    orc = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, mode, k, 1 if cache else 0,
                                 wl.S, cap, cell=cell), m)
    return eng, orc


@pytest.mark.parametrize("mode,k", [(KEY_SIGN, 0), (KEY_ROUND, 2), (KEY_OFF, 0)])
def test_tiny_config_all_frames(mode, k):
    """configs[0]: V 1k, E=H=64, 2^16 3-gram, 32 queries x 100 frames, fp32."""
    d, m = model("tiny")
    wl = generate_workload(1, 100, 32, d.V, seed=7)
    eng, orc = pair(d, m, wl, mode, k)
    rep = replay_compare(eng, orc, wl, tol_score=1e-5, tol_state=1e-5)
    assert rep["miss"] > 100 and rep["qhit"] > 1000


def test_tiny_cache_disabled():
    d, m = model("tiny")
    wl = generate_workload(1, 30, 32, d.V, seed=8)
    eng, orc = pair(d, m, wl, KEY_SIGN, 0, cache=False)
    rep = replay_compare(eng, orc, wl)
    assert rep["miss"] == wl.n_total


def forgetful_model(H=16, E=16, V=64, seed=5):
    """Input-dominated GRU (z ~ 0.98, tiny recurrent weights): a state is almost
    a function of its last word, so histories that end in the same word get
    equal lossy keys and the hidden cache's SHIT paths are exercised."""
    d = ModelDims(V=V, E=E, H=H, maxent_log2=10, N=4)
    m = generate_model(d, seed=seed, scale=1.0, bf16_grid=False)
    for k in ("Uz", "Ur", "Uh"):
        m[k] = (m[k] * 0.02).astype(np.float32)
    m["bz"] = np.full(H, 4.0, np.float32)
    return d, m


@pytest.mark.parametrize("mode,k", [(KEY_SIGN, 0), (KEY_ROUND, 1), (KEY_ROUND, 2), (KEY_OFF, 0)])
def test_lossy_hidden_hits_multisession(mode, k):
    """Many SHITs (earlier-call and same-call owners), 3 sessions, fp32 path."""
    d, m = forgetful_model()
    wl = generate_workload(3, 40, 96, d.V, seed=21, dur=(2, 6))
    eng, orc = pair(d, m, wl, mode, k)
    rep = replay_compare(eng, orc, wl)
    assert rep["shit"] >= {KEY_SIGN: 100, KEY_ROUND: 20, KEY_OFF: 0}[mode], rep


def test_moderate_config_prefix():
    """configs[1]: V 100k, H 256, 2^22 4-gram, 256 queries/frame (first 60 frames)."""
    d, m = model("moderate")
    wl = generate_workload(1, 60, 256, d.V, seed=7)
    for mode in (KEY_OFF, KEY_SIGN):
        eng, orc = pair(d, m, wl, mode)
        rep = replay_compare(eng, orc, wl)
        assert rep["miss"] > 100


def test_large_config_fp32_prefix():
    """configs[2] shapes: V 200k, H 1024, 2^27 4-gram, 2,048 queries/frame, fp32 path."""
    d, m = model("large")
    wl = generate_workload(1, 3, 2048, d.V, seed=7)
    eng, orc = pair(d, m, wl, KEY_SIGN)
    replay_compare(eng, orc, wl)


def test_multisession_config_sample():
    """configs[4] shapes: 4 of the 64 sessions x 2,048 queries/frame, large model."""
    d, m = model("large")
    wl = generate_workload(4, 2, 2048, d.V, seed=7)
    eng, orc = pair(d, m, wl, KEY_SIGN)
    replay_compare(eng, orc, wl)


def test_edge_cases_invalid_and_ragged():
    d, m = model("tiny")
    eng = RNNLM.from_dims(d, m, key_mode=KEY_SIGN, num_sessions=2, max_queries_per_call=1000,
                          max_histories_per_session=64)
    orc = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_SIGN, 0, 1, 2, 64), m)
    # empty batch
    e = torch.empty(0, dtype=torch.int32, device="cuda")
    eng.query_batch(e, e, e)
    frames = [
        # session, parent, word: dup pairs, word >= V, parent unborn, session >= S
        ([0, 0, 0, 0, 1, 1, 1, 2], [0, 0, 0, 5, 0, 0, 0, 0], [3, 3, 1000, 4, 7, 7, 2, 1]),
        ([0] * 5 + [1] * 3, [1, 2, 1, 1, 2, 1, 2, 2], [9, 9, 9, 8, 9, 3, 4, 4]),
    ]
    for sess, par, wrd in frames:
        sc, ch, oc = eng.query_batch(_dev(sess), _dev(par), _dev(wrd))
        osc, och, ooc = orc.query_frame(sess, par, wrd)
        assert np.array_equal(oc.cpu().numpy(), ooc)
        assert np.array_equal(ch.cpu().numpy().view(np.uint32), och)
        v = ooc != O.INVALID
        assert np.max(np.abs(sc.cpu().numpy()[v] - osc[v])) <= 1e-5
        assert np.all(np.isnan(sc.cpu().numpy()[~v]))
    st = eng.cache_stats()
    ost = orc.stats()
    for kk in ("total_queries", "query_hits", "hidden_lookups", "hidden_hits", "gru_computations"):
        assert st[kk] == ost[kk]
    assert st["sticky_error"] != 0
    # a ragged batch of 1000 queries (not a multiple of the 1024-query scan tile / 256 threads)
    rng = np.random.default_rng(3)
    sess = np.sort(rng.integers(0, 2, 1000))
    par = np.zeros(1000)
    wrd = rng.integers(0, d.V, 1000)
    sc, ch, oc = eng.query_batch(_dev(sess), _dev(par), _dev(wrd))
    osc, och, ooc = orc.query_frame(sess, par, wrd)
    assert np.array_equal(oc.cpu().numpy(), ooc)
    assert np.array_equal(ch.cpu().numpy().view(np.uint32), och)   # includes capacity overflow


def test_unsorted_batch_rejected():
    d, m = model("tiny")
    eng = RNNLM.from_dims(d, m, num_sessions=2, max_queries_per_call=8, max_histories_per_session=64)
    sc, ch, oc = eng.query_batch(_dev([1, 0]), _dev([0, 0]), _dev([1, 2]))
    assert set(oc.cpu().numpy().tolist()) == {INVALID}
    assert eng.cache_stats()["sticky_error"] == 1
    assert eng.cache_stats()["total_queries"] == 0


def test_mode_off_equals_cache_disabled_bitwise():
    """Cache-hit equivalence on the GPU: with a lossless key the cached run
    returns exactly what direct evaluation returns (BASELINE north_star)."""
    d, m = model("tiny")
    wl = generate_workload(2, 40, 32, d.V, seed=9)
    outs = []
    for cache in (True, False):
        eng = RNNLM.from_dims(d, m, key_mode=KEY_OFF, cache_enabled=cache, num_sessions=2,
                              max_queries_per_call=64, max_histories_per_session=4096)
        child = np.zeros(wl.n_total, np.uint32)
        scores = np.zeros(wl.n_total, np.float32)
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            par = O.resolve_parents(wl.parent_ref[sl], child)
            sc, ch, _ = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
            child[sl] = ch.cpu().numpy().view(np.uint32)
            scores[sl] = sc.cpu().numpy()
        states = [eng.read_states(s, child[wl.session == s]).cpu().numpy() for s in range(2)]
        outs.append((scores, states))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("mode,k", [(KEY_SIGN, 0), (KEY_ROUND, 1), (KEY_ROUND, 2), (KEY_ROUND, 3),
                                    (KEY_ROUND, 4), (KEY_OFF, 0)])
def test_compression_kernel_bit_exact(mode, k):
    """(a1) keys bit-exact vs the oracle on random and adversarial vectors."""
    H = 64
    d = ModelDims(V=4, E=8, H=H, maxent_log2=4, N=2)
    _, m = model(d, seed=3)
    eng = RNNLM.from_dims(d, m, key_mode=mode, round_digits=k, max_queries_per_call=4,
                          max_histories_per_session=8)
    rng = np.random.default_rng(k + 10 * mode)
    rows = [rng.uniform(-1, 1, (4000, H)), rng.uniform(-1e-3, 1e-3, (500, H))]
    # ties n.5 / 10^k on exactly representable values, zeros of both signs, near +-1
    ties = np.array([0.125, -0.125, 0.375, -0.375, 0.5, -0.5, 0.0, -0.0, 0.25, -0.25, 0.05,
                     -0.005, 0.0005, -0.00005, 0.99995, -0.99995], dtype=np.float32)
    rows.append(np.tile(ties, (8, H // len(ties))))
    rows.append(rng.choice([-1, 1], (100, H)) * np.nextafter(np.float32(1), np.float32(0)))
    X = np.concatenate(rows).astype(np.float32)
    got = eng.encode_states(torch.from_numpy(X)).cpu().numpy()
    for i in range(len(X)):
        assert np.array_equal(got[i], O.compress(X[i], mode, k)), (i, X[i][:4])


def test_maxent_indices_bit_exact():
    d, m = model("moderate")
    wl = generate_workload(1, 30, 256, d.V, seed=4)
    eng, orc = pair(d, m, wl, KEY_SIGN)
    replay_compare(eng, orc, wl, check_codes=False)
    rng = np.random.default_rng(0)
    h, _ = orc.num_handles(0)
    par = rng.integers(0, h, 3000).astype(np.uint32)
    wrd = rng.integers(0, d.V, 3000).astype(np.uint32)
    got = eng.maxent_indices(_dev(np.zeros(3000)), _dev(par), _dev(wrd)).cpu().numpy().view(np.uint64)
    ctxs = orc.read_ctx(0, par)
    for i in range(3000):
        ref = O.maxent_indices(ctxs[i], int(wrd[i]), d.N, d.M)
        assert got[i][:len(ref)].tolist() == ref
        assert all(x == 2 ** 64 - 1 for x in got[i][len(ref):])


def test_deterministic_rerun():
    d, m = forgetful_model()
    wl = generate_workload(3, 25, 96, d.V, seed=22, dur=(2, 6))
    runs = []
    for _ in range(2):
        eng = RNNLM.from_dims(d, m, key_mode=KEY_SIGN, num_sessions=3, max_queries_per_call=wl.n_per_frame,
                              max_histories_per_session=wl.max_histories_hint())
        child = np.zeros(wl.n_total, np.uint32)
        out = []
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            par = O.resolve_parents(wl.parent_ref[sl], child)
            sc, ch, oc = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
            child[sl] = ch.cpu().numpy().view(np.uint32)
            out.append((sc.cpu().numpy().view(np.uint32), child[sl].copy(), oc.cpu().numpy()))
        runs.append(out)
    for a, b in zip(*runs):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_resolve_parents_kernel():
    from paper_1801_09866_b200 import resolve_parents
    ref = torch.tensor([-1, 0, 2, 1], dtype=torch.int64, device="cuda")
    log = torch.tensor([7, 8, 9], dtype=torch.int32, device="cuda")
    out = torch.empty(4, dtype=torch.int32, device="cuda")
    resolve_parents(ref, log, out)
    assert out.cpu().tolist() == [0, 7, 9, 8]


# ---------------------------------------------------------------- BF16 tensor-core path (tcgen05)
@pytest.mark.parametrize("mode", [KEY_OFF, KEY_SIGN])
def test_moderate_bf16_tensor_core(mode):
    d, m = model("moderate")
    wl = lattice(1, 40, 256, d.V, seed=17)
    eng, orc = pair(d, m, wl, mode, math=MATH_BF16)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[MATH_BF16], tol_state=TOL[MATH_BF16])
    assert rep["miss"] > 300


@pytest.mark.parametrize("k", [1, 2, 3])
def test_moderate_bf16_round_codes(k):
    """round:k keys (int8 codes for k <= 2, int16 for k = 3) are encoded inside
    the tcgen05 phase-2 epilogue; codes bit-exact vs the oracle's compress() of
    the same GPU vector, lossy hidden-cache hits identical (replay protocol)."""
    d, m = model("moderate")
    wl = lattice(1, 40, 256, d.V, seed=19)
    eng, orc = pair(d, m, wl, KEY_ROUND, k=k, math=MATH_BF16)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[MATH_BF16], tol_state=TOL[MATH_BF16])
    assert rep["miss"] > 300


@pytest.mark.parametrize("lag", ["2", "6"])
def test_bf16_interleaved_phase_schedule(lag, monkeypatch):
    """Phase-2 tiles interleaved with the phase-1 tiles of later M-tiles (the
    middle section of the tile order, RNNLM_TC_LAG smaller than the number of
    M-tiles): both bf16 kernels, 4,000 rows = 16 pair / 32 single M-tiles."""
    if lag:
        monkeypatch.setenv("RNNLM_TC_LAG", lag)
    d, m = model("large")
    wl = generate_workload(2, 2, 2000, d.V, seed=23)
    for pk, p2n in (("1", None), ("1", "0"), ("0", None)):
        monkeypatch.setenv("RNNLM_TC_PAIR", pk)
        if p2n is not None:     # 256-unit phase-2 tiles (the large-call instance)
            monkeypatch.setenv("RNNLM_TC_P2N_MAX", p2n)
        else:
            monkeypatch.delenv("RNNLM_TC_P2N_MAX", raising=False)
        eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16, cache=False)
        rep = replay_compare(eng, orc, wl, tol_score=TOL[MATH_BF16], tol_state=TOL[MATH_BF16])
        assert rep["miss"] == wl.n_total


@pytest.mark.parametrize("pair_kernel", ["1", "0"])
@pytest.mark.parametrize("shape", ["full", "ragged_multisession"])
def test_bf16_cta_pair_kernel(shape, pair_kernel, monkeypatch):
    """Both bf16 GRU kernels against the oracle: the CTA pair (cta_group::2,
    M = 256; the default, RNNLM_TC_PAIR=1) and one CTA per tile
    (RNNLM_TC_PAIR=0): full 256-row pair tiles and a ragged multi-session batch."""
    monkeypatch.setenv("RNNLM_TC_PAIR", pair_kernel)
    d, m = model("large")
    if shape == "full":
        wl = generate_workload(1, 2, 2048, d.V, seed=5)
        eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16, cache=False)
        rep = replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)
        assert rep["miss"] == wl.n_total
    else:
        wl = generate_workload(3, 3, 300, d.V, seed=6)
        eng, orc = pair(d, m, wl, KEY_ROUND, k=2, math=MATH_BF16)
        replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)


@pytest.mark.parametrize("math", [MATH_BF16, MATH_BF16X3])
@pytest.mark.parametrize("p2n_max", ["0", None])
def test_cta_pair_phase2_tile_widths(math, p2n_max, monkeypatch):
    """The CTA-pair kernel's two phase-2 tile shapes against the oracle:
    256-unit tiles (RNNLM_TC_P2N_MAX=0: the instance calls of more than 32k
    queries run) and 128-unit tiles (the default for these small calls).
    All-miss full tiles, then a ragged multi-session batch with round keys."""
    monkeypatch.setenv("RNNLM_TC_PAIR", "1")
    if p2n_max is not None:
        monkeypatch.setenv("RNNLM_TC_P2N_MAX", p2n_max)
    tol = TOL[math]
    d, m = model("large")
    wl = generate_workload(1, 2, 2048, d.V, seed=5)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=math, cache=False)
    rep = replay_compare(eng, orc, wl, tol_score=tol, tol_state=tol)
    assert rep["miss"] == wl.n_total
    wl = generate_workload(3, 3, 300, d.V, seed=6)
    eng, orc = pair(d, m, wl, KEY_ROUND, k=2, math=math)
    replay_compare(eng, orc, wl, tol_score=tol, tol_state=tol)


def test_large_bf16_cache_off_full_tiles():
    """All-miss stress: 2,048 GRU rows per frame = 16 full M-tiles + ragged frames."""
    d, m = model("large")
    wl = generate_workload(1, 2, 2048, d.V, seed=5)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16, cache=False)
    rep = replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)
    assert rep["miss"] == wl.n_total


def test_large_bf16_ragged_rows():
    """Q not a multiple of 128 (ragged last M-tile) on the large model."""
    d, m = model("large")
    wl = generate_workload(1, 2, 300, d.V, seed=6)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16, cache=False)
    replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)


def test_multisession_bf16_sample():
    d, m = model("large")
    wl = generate_workload(4, 3, 2048, d.V, seed=7)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16)
    replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)


# ---------------------------------------------------------------- TF32 tensor-core path (tcgen05 kind::tf32)
@pytest.mark.parametrize("mode", [KEY_OFF, KEY_SIGN])
def test_moderate_tf32_tensor_core(mode):
    d, m = model("moderate")
    wl = lattice(1, 40, 256, d.V, seed=17)
    eng, orc = pair(d, m, wl, mode, math=MATH_TF32)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[MATH_TF32], tol_state=TOL[MATH_TF32])
    assert rep["miss"] > 300


def test_large_tf32_cache_off_full_tiles():
    d, m = model("large")
    wl = generate_workload(1, 2, 2048, d.V, seed=5)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_TF32, cache=False)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[MATH_TF32], tol_state=TOL[MATH_TF32])
    assert rep["miss"] == wl.n_total


def test_large_tf32_ragged_multisession():
    d, m = model("large")
    wl = generate_workload(3, 3, 300, d.V, seed=6)
    eng, orc = pair(d, m, wl, KEY_ROUND, k=2, math=MATH_TF32)
    replay_compare(eng, orc, wl, tol_score=TOL[MATH_TF32], tol_state=TOL[MATH_TF32])


def test_tf32_more_accurate_than_bf16():
    """TF32 operands keep 11 significant bits (bf16: 8), so with weights that
    are NOT on the bf16 grid the TF32 path's state error vs the fp64 oracle is
    several times below the bf16 path's on the same rows (replay mode)."""
    d = ModelDims(V=1000, E=256, H=256, maxent_log2=16, N=3)
    m = generate_model(d, seed=3, scale=0.1, bf16_grid=False)
    wl = generate_workload(1, 6, 256, d.V, seed=8)
    errs = {}
    for math in (MATH_BF16, MATH_TF32):
        eng, orc = pair(d, m, wl, KEY_SIGN, math=math, cache=False)
        errs[math] = replay_compare(eng, orc, wl, tol_score=1e-2, tol_state=1e-2)["max_state_err"]
    assert errs[MATH_TF32] < 0.3 * errs[MATH_BF16], errs
    assert errs[MATH_TF32] < 1e-4, errs


def test_per_query_calls_equal_per_frame_batches():
    """Frame-wise batching changes nothing in the results: one call
    per query returns bitwise the same scores, handles and states."""
    d, m = forgetful_model()
    wl = generate_workload(2, 12, 24, d.V, seed=31, dur=(2, 6))
    outs = []
    for per_query in (False, True):
        eng = RNNLM.from_dims(d, m, key_mode=KEY_SIGN, num_sessions=2, max_queries_per_call=64,
                              max_histories_per_session=wl.max_histories_hint())
        child = np.zeros(wl.n_total, np.uint32)
        score = np.zeros(wl.n_total, np.float32)
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            par = O.resolve_parents(wl.parent_ref[sl], child)
            if per_query:
                for i in range(sl.start, sl.stop):
                    j = i - sl.start
                    sc, ch, _ = eng.query_batch(_dev(wl.session[i:i + 1]), _dev(par[j:j + 1]),
                                                _dev(wl.word[i:i + 1]))
                    child[i] = ch.cpu().numpy().view(np.uint32)[0]
                    score[i] = sc.cpu().numpy()[0]
            else:
                sc, ch, _ = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
                child[sl] = ch.cpu().numpy().view(np.uint32)
                score[sl] = sc.cpu().numpy()
        states = [eng.read_states(s, child[wl.session == s]).cpu().numpy() for s in range(2)]
        outs.append((score, child, states, eng.cache_stats()))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1], outs[1][1])
    for a, b in zip(outs[0][2], outs[1][2]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert outs[0][3]["gru_computations"] == outs[1][3]["gru_computations"]


# ---------------------------------------------------------------- cell variant GRU_LBR
@pytest.mark.parametrize("math", [MATH_FP32, MATH_BF16, MATH_TF32])
def test_lbr_cell_moderate(math):
    """Linear-before-reset cell on every math path: FP32 SIMT (phase 1 keeps r,
    phase 2 contracts h), BF16 / TF32 one-phase tcgen05 tiles (N = 192 over
    the x part, N = 128 + 64 over the h part)."""
    d, m = model("moderate")
    wl = lattice(1, 30, 256, d.V, seed=23)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=math, cell=O.CELL_GRU_LBR)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math])
    assert rep["miss"] > 200


def test_lbr_cell_large_full_tiles_and_round_codes():
    """Large model, all-miss (16 full M-tiles, 16 unit tiles each) and a ragged
    multi-session round:2 batch, LBR on the bf16 tensor-core path."""
    d, m = model("large")
    wl = generate_workload(1, 2, 2048, d.V, seed=5)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16, cache=False, cell=O.CELL_GRU_LBR)
    rep = replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)
    assert rep["miss"] == wl.n_total
    wl = generate_workload(3, 3, 300, d.V, seed=6)
    eng, orc = pair(d, m, wl, KEY_ROUND, k=2, math=MATH_BF16, cell=O.CELL_GRU_LBR)
    replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)


def test_lbr_differs_from_gru():
    """The two cells are different functions (same weights, same stream):
    children of the root agree (h = 0 makes both recurrent terms vanish),
    deeper histories do not."""
    d, m = model("moderate")
    wl = generate_workload(1, 30, 64, d.V, seed=29)
    outs = []
    for cell in (0, O.CELL_GRU_LBR):
        eng, _ = pair(d, m, wl, KEY_OFF, math=MATH_FP32, cell=cell)
        child = np.zeros(wl.n_total, np.uint32)
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            par = O.resolve_parents(wl.parent_ref[sl], child)
            _, ch, _ = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
            child[sl] = ch.cpu().numpy().view(np.uint32)
        last = int(child.max())
        outs.append(eng.read_states(0, np.arange(last - 7, last + 1, dtype=np.uint32)).cpu().numpy())
    assert np.max(np.abs(outs[0] - outs[1])) > 1e-4


# ---------------------------------------------------------------- offline level batching
@pytest.mark.parametrize("path", [GRU_TILES, GRU_GEMV])
@pytest.mark.parametrize("math", [MATH_BF16, MATH_FP32])
def test_offline_level_batches_equal_online(math, path):
    """The same utterances run level by level (paper_1801_09866_b200.offline)
    instead of frame by frame: with lossless keys every query gets bitwise the
    same score and its child bitwise the same state (batch-invariant kernels;
    both schedules on the same GRU kernels -- tiles or GEMV)."""
    from paper_1801_09866_b200.offline import OfflineRunner
    d, m = model("moderate")
    wl = generate_workload(2, 40, 128, d.V, seed=43)
    cap = wl.max_histories_hint()
    mk = lambda B: RNNLM.from_dims(d, m, key_mode=KEY_OFF, math=math, num_sessions=wl.S,
                                   max_queries_per_call=B, max_histories_per_session=cap, gru_path=path)
    on = mk(wl.n_per_frame)
    child_on = np.zeros(wl.n_total, np.uint32)
    score_on = np.zeros(wl.n_total, np.float32)
    for t in range(wl.frames):
        sl = wl.frame_slice(t)
        par = O.resolve_parents(wl.parent_ref[sl], child_on)
        sc, ch, _ = on.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
        score_on[sl] = sc.cpu().numpy()
        child_on[sl] = ch.cpu().numpy().view(np.uint32)
    off = mk(4096)
    runner = OfflineRunner(off, wl, max_batch=4096)
    sc, ch = runner.run()
    assert len(runner.batches) < wl.frames
    assert np.array_equal(score_on.view(np.uint32), sc.cpu().numpy().view(np.uint32))
    child_off = ch.cpu().numpy().view(np.uint32)
    for s in range(wl.S):
        msk = wl.session == s
        a = on.read_states(s, child_on[msk]).cpu().numpy()
        b = off.read_states(s, child_off[msk]).cpu().numpy()
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("math", [MATH_FP32, MATH_BF16, MATH_TF32])
def test_rnn_cell_moderate(math):
    """Vanilla-RNN cell (h' = sigma(Wh x + Uh h + bh)) on every math
    path: FP32 SIMT (phase 2 contracts h), BF16 / TF32 one-phase tcgen05 tiles
    of A1 x [Wh | Uh]; lossy sign keys, codes bit-exact."""
    d, m = model("moderate")
    wl = lattice(1, 30, 256, d.V, seed=31)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=math, cell=O.CELL_RNN)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math])
    # logistic states are all positive: every sign code is all ones, so a
    # word's later queries all merge with its first (many SHITs, few MISSes)
    assert rep["miss"] > 50 and rep["shit"] > 100


def test_rnn_cell_large_full_tiles():
    d, m = model("large")
    wl = generate_workload(1, 2, 2048, d.V, seed=5)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16, cache=False, cell=O.CELL_RNN)
    rep = replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)
    assert rep["miss"] == wl.n_total


# ---------------------------------------------------------------- the hidden sizes of the paper's Fig. 4
@pytest.mark.parametrize("H", [128, 512])
@pytest.mark.parametrize("cell", [0, O.CELL_GRU_LBR, O.CELL_RNN])
@pytest.mark.parametrize("math", [MATH_BF16, MATH_TF32])
def test_fig4_hidden_sizes_tensor_core(H, cell, math):
    """H = 128 (phase-2 / RNN tiles narrow to 128 units, N = 128) and H = 512 on
    the tensor-core paths, every cell, E = H, lossy sign keys."""
    d = ModelDims(V=5000, E=H, H=H, maxent_log2=18, N=4)
    m = generate_model(d, seed=77)
    wl = lattice(1, 20, 300, d.V, seed=13)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=math, cell=cell)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math])
    assert rep["miss"] > (30 if cell == O.CELL_RNN else 100)   # RNN: positive states, sign codes merge


@pytest.mark.parametrize("pair_kernel", ["1", "0"])
@pytest.mark.parametrize("E", [64, 192, 448])
@pytest.mark.parametrize("math", [MATH_BF16, MATH_TF32])
def test_tensor_core_embed_neq_hidden(E, math, pair_kernel, monkeypatch):
    """E != H on the tensor-core paths (H = 256): the A1 gather's x and h row
    chunks of different lengths (E/8 vs H/8 16-byte words), K = E + H not a
    multiple of 256, both bf16 kernels."""
    if math == MATH_TF32 and pair_kernel == "1":
        pytest.skip("TF32 runs the one-CTA kernel only")
    monkeypatch.setenv("RNNLM_TC_PAIR", pair_kernel)
    d = ModelDims(V=3000, E=E, H=256, maxent_log2=16, N=3)
    m = generate_model(d, seed=41)
    wl = lattice(2, 14, 300, d.V, seed=19)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=math)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math])
    assert rep["miss"] > 100


# ---------------------------------------------------------------- 3xTF32: fp32-accurate tensor-core GRU
def test_tf32x3_moderate_fp32_tolerance():
    """RNNLM_MATH_TF32X3 holds the FP32 path's 1e-5 bar on scores and states
    (operands split into TF32 hi + lo parts, three products), sign keys with
    lossy hits, codes bit-exact."""
    d, m = model("moderate")
    wl = lattice(1, 30, 256, d.V, seed=17)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_TF32X3)
    rep = replay_compare(eng, orc, wl, tol_score=1e-5, tol_state=1e-5)
    assert rep["miss"] > 200


def test_tf32x3_large_full_tiles_and_ragged():
    d, m = model("large")
    wl = generate_workload(1, 2, 2048, d.V, seed=5)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_TF32X3, cache=False)
    rep = replay_compare(eng, orc, wl, tol_score=1e-5, tol_state=1e-5)
    assert rep["miss"] == wl.n_total
    wl = generate_workload(3, 3, 300, d.V, seed=6)
    eng, orc = pair(d, m, wl, KEY_ROUND, k=2, math=MATH_TF32X3)
    replay_compare(eng, orc, wl, tol_score=1e-5, tol_state=1e-5)


def test_tf32x3_off_grid_weights_accuracy():
    """Weights NOT on the bf16 grid: the 3xTF32 states sit at FP32-path error
    (< 1e-5 from the fp64 oracle), far below single TF32."""
    d = ModelDims(V=1000, E=256, H=256, maxent_log2=16, N=3)
    m = generate_model(d, seed=3, scale=0.1, bf16_grid=False)
    wl = generate_workload(1, 6, 256, d.V, seed=8)
    errs = {}
    for math in (MATH_TF32, MATH_TF32X3):
        eng, orc = pair(d, m, wl, KEY_SIGN, math=math, cache=False)
        errs[math] = replay_compare(eng, orc, wl, tol_score=1e-2, tol_state=1e-2)["max_state_err"]
    assert errs[MATH_TF32X3] < 1e-5, errs
    assert errs[MATH_TF32X3] < 0.1 * errs[MATH_TF32], errs


def test_results_ready_before_state_update():
    """rnnlm_results_ready: a second stream that waits only for it and copies
    the scores / handles out sees the final values (the large model's GRU may
    still be running), identical to the values after a full synchronize."""
    d, m = model("large")
    wl = generate_workload(4, 3, 1024, d.V, seed=9)
    eng, _ = pair(d, m, wl, KEY_SIGN, math=MATH_BF16)
    child = np.zeros(wl.n_total, np.uint32)
    side = torch.cuda.Stream()
    for t in range(wl.frames):
        sl = wl.frame_slice(t)
        par = O.resolve_parents(wl.parent_ref[sl], child)
        sc = torch.empty(wl.n_per_frame, dtype=torch.float32, device="cuda")
        ch = torch.empty(wl.n_per_frame, dtype=torch.int32, device="cuda")
        eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]), score=sc, child=ch)
        eng.results_ready(stream=side)
        with torch.cuda.stream(side):
            early_sc = sc.to("cpu", non_blocking=True)
            early_ch = ch.to("cpu", non_blocking=True)
        side.synchronize()
        torch.cuda.synchronize()
        assert np.array_equal(early_sc.numpy().view(np.uint32), sc.cpu().numpy().view(np.uint32))
        assert np.array_equal(early_ch.numpy(), ch.cpu().numpy())
        child[sl] = ch.cpu().numpy().view(np.uint32)


def test_tf32x3_skips_zero_weight_lo_segment(monkeypatch):
    """bf16-grid weights and embeddings are TF32-exact, so the 3xTF32 A_hi.W_lo
    product and A_lo.W_hi over the embedding part of K are identically zero
    and are skipped (1.5 products per MAC at E = H); running them anyway
    (RNNLM_SPLIT_ALL_SEGMENTS) only adds exact zeros: bitwise the same scores
    and states.  Off-grid weights keep all three."""
    d, m = model("moderate")
    wl = lattice(1, 12, 256, d.V, seed=5)
    outs = []
    for allseg in (False, True):
        if allseg:
            monkeypatch.setenv("RNNLM_SPLIT_ALL_SEGMENTS", "1")
        eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_TF32X3)
        assert eng.tf32x3_products() == (3.0 if allseg else 1.5)   # E = H: (K + H) / K
        child = np.zeros(wl.n_total, np.uint32)
        score = np.zeros(wl.n_total, np.float32)
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            par = O.resolve_parents(wl.parent_ref[sl], child)
            s_, c_, _ = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
            score[sl], child[sl] = s_.cpu().numpy(), c_.cpu().numpy().view(np.uint32)
        outs.append((score, eng.read_states(0, child).cpu().numpy()))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1].view(np.uint32), outs[1][1].view(np.uint32))
    monkeypatch.delenv("RNNLM_SPLIT_ALL_SEGMENTS")
    d2 = ModelDims(V=1000, E=256, H=256, maxent_log2=16, N=3)
    m2 = generate_model(d2, seed=3, scale=0.1, bf16_grid=False)
    eng2 = RNNLM.from_dims(d2, m2, math=MATH_TF32X3, max_queries_per_call=8, max_histories_per_session=8)
    assert eng2.tf32x3_products() == 3.0


# ---------------------------------------------------------------- BF16X3: fp32-accurate on the bf16 tensor cores
@pytest.mark.parametrize("pair_kernel", ["1", "0"])
def test_bf16x3_moderate_fp32_tolerance(pair_kernel, monkeypatch):
    """RNNLM_MATH_BF16X3 holds the FP32 path's 1e-5 bar on scores and states
    (activations split into three bf16 parts), sign keys with lossy hits,
    codes bit-exact; the CTA pair and one CTA per tile."""
    monkeypatch.setenv("RNNLM_TC_PAIR", pair_kernel)
    d, m = model("moderate")
    wl = lattice(1, 30, 256, d.V, seed=17)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16X3)
    rep = replay_compare(eng, orc, wl, tol_score=1e-5, tol_state=1e-5)
    assert rep["miss"] > 200


@pytest.mark.parametrize("pair_kernel", ["1", "0"])
def test_bf16x3_large_full_tiles_and_ragged(pair_kernel, monkeypatch):
    monkeypatch.setenv("RNNLM_TC_PAIR", pair_kernel)
    d, m = model("large")
    wl = generate_workload(1, 2, 2048, d.V, seed=5)
    eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16X3, cache=False)
    rep = replay_compare(eng, orc, wl, tol_score=1e-5, tol_state=1e-5)
    assert rep["miss"] == wl.n_total
    wl = generate_workload(3, 3, 300, d.V, seed=6)
    eng, orc = pair(d, m, wl, KEY_ROUND, k=2, math=MATH_BF16X3)
    replay_compare(eng, orc, wl, tol_score=1e-5, tol_state=1e-5)


@pytest.mark.parametrize("pair_kernel", ["1", "0"])
def test_bf16x3_off_grid_weights_accuracy(pair_kernel, monkeypatch):
    """Weights and embeddings NOT on the bf16 grid: all six products run, the
    states sit at FP32-path error (< 1e-5 from the fp64 oracle), far below
    plain bf16 operands."""
    monkeypatch.setenv("RNNLM_TC_PAIR", pair_kernel)
    d = ModelDims(V=1000, E=256, H=256, maxent_log2=16, N=3)
    m = generate_model(d, seed=3, scale=0.1, bf16_grid=False)
    wl = generate_workload(1, 6, 256, d.V, seed=8)
    errs = {}
    for math in (MATH_BF16, MATH_BF16X3):
        eng, orc = pair(d, m, wl, KEY_SIGN, math=math, cache=False)
        if math == MATH_BF16X3:
            assert eng.tf32x3_products() == 6.0
        errs[math] = replay_compare(eng, orc, wl, tol_score=1e-1, tol_state=1e-1)["max_state_err"]
    assert errs[MATH_BF16X3] < 1e-5, errs
    assert errs[MATH_BF16X3] < 0.01 * errs[MATH_BF16], errs


def test_bf16x3_skips_zero_segments(monkeypatch):
    """bf16-grid weights and embeddings: the products with a zero weight part
    and, over the embedding part of K, with a zero embedding part are skipped
    (2 bf16 products per MAC at E = H: x_hi.W over E, h_hi/mid/lo.W over H);
    running all six anyway (RNNLM_SPLIT_ALL_SEGMENTS) only adds exact zeros:
    bitwise the same scores and states."""
    d, m = model("moderate")
    wl = lattice(1, 12, 256, d.V, seed=5)
    outs = []
    for allseg in (False, True):
        if allseg:
            monkeypatch.setenv("RNNLM_SPLIT_ALL_SEGMENTS", "1")
        eng, orc = pair(d, m, wl, KEY_SIGN, math=MATH_BF16X3)
        assert eng.tf32x3_products() == (6.0 if allseg else 2.0)   # E = H: (E + 3H) / (E + H)
        child = np.zeros(wl.n_total, np.uint32)
        score = np.zeros(wl.n_total, np.float32)
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            par = O.resolve_parents(wl.parent_ref[sl], child)
            s_, c_, _ = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
            score[sl], child[sl] = s_.cpu().numpy(), c_.cpu().numpy().view(np.uint32)
        outs.append((score, eng.read_states(0, child).cpu().numpy()))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1].view(np.uint32), outs[1][1].view(np.uint32))
