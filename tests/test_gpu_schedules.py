"""GPU vs ORACLE under the two alternative call schedules of SURVEY 8(f):

* (f1) one call per query -- the paper's per-query transfer mode (P:181-184,
  Table 2): the same queries, each its own rnnlm_query_batch call;
* (f4) offline level batching (paper_1801_09866_b200.offline): the
  whole stream grouped by dependency level, several frames per call.

Both sides make the same calls (tests/parity_util.replay_compare with
``batches``), so every decision -- including which query is a lossy key's
first occupant, which depends on the schedule -- must be bit-identical to the
oracle, at every key mode; states / scores within the path's tolerance.
"""
import numpy as np
import pytest

from paper_1801_09866_b200 import GRU_GEMV, GRU_TILES, KEY_OFF, KEY_ROUND, KEY_SIGN, MATH_BF16, MATH_FP32, MATH_TF32
from paper_1801_09866_b200.offline import level_schedule
from synth import generate_workload
from tests.parity_util import replay_compare
from tests.test_gpu_parity import TOL, forgetful_model, model, pair

pytestmark = pytest.mark.gpu

MODES = [(KEY_OFF, 0), (KEY_SIGN, 0), (KEY_ROUND, 1), (KEY_ROUND, 2), (KEY_ROUND, 3)]


@pytest.mark.parametrize("mode,k", MODES)
@pytest.mark.parametrize("math", [MATH_FP32, MATH_BF16])
def test_per_query_calls_vs_oracle(math, mode, k):
    """(f1): one call per query; the forgetful model makes lossy keys merge."""
    if math == MATH_FP32:
        d, m = forgetful_model()
    else:                                     # tensor-core tiles need E % 64, H % 128
        d, m = model("moderate")
    wl = generate_workload(2, 20, 32, d.V, seed=31, dur=(2, 6), eps=0.3, beam_scale=4)
    eng, orc = pair(d, m, wl, mode, k=k, math=math, B=64)
    batches = [np.array([i]) for i in range(wl.n_total)]
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math], batches=batches)
    assert rep["frames"] == wl.n_total and rep["miss"] > 100
    if math == MATH_FP32 and mode != KEY_OFF and k < 3:   # oracle: sign 97, round:1 43, round:2 26
        assert rep["shit"] > 15, rep


@pytest.mark.parametrize("mode,k", MODES)
@pytest.mark.parametrize("math", [MATH_FP32, MATH_BF16, MATH_TF32])
def test_offline_level_batches_vs_oracle(math, mode, k):
    """(f4): level-batched calls (several frames' queries per call, sessions
    mixed), lossy keys merging (H = 256 model, lattice stream)."""
    d, m = model("moderate")
    wl = generate_workload(2, 120, 128, d.V, seed=13, dur=(2, 6), eps=0.1)
    batches = level_schedule(wl.session, wl.parent_ref, wl.frame_ptr, max_batch=2048)
    assert len(batches) < wl.frames
    eng, orc = pair(d, m, wl, mode, k=k, math=math, B=2048)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math], batches=batches)
    assert rep["miss"] > 500
    if (mode, k) in ((KEY_SIGN, 0), (KEY_ROUND, 1), (KEY_ROUND, 2)):   # oracle: 1250, 772, 221
        assert rep["shit"] > 50, rep


@pytest.mark.parametrize("math", [MATH_FP32, MATH_BF16])
def test_graph_replay_equals_direct_calls(math):
    """rnnlm_graph_create / rnnlm_graph_launch: one captured call replayed per
    frame on fixed buffers, with the frame's query count read on the device
    (staggered sessions make the frame sizes vary), returns bitwise what
    rnnlm_query_batch returns; stats equal."""
    import torch
    import oracle as O
    from tests.parity_util import _dev
    d, m = model("moderate")
    wl = generate_workload(3, 90, 64, d.V, seed=11, dur=(2, 5), eps=0.1).staggered([0, 7, 19])
    B = wl.n_per_frame
    outs = []
    for use_graph in (False, True):
        eng, _ = pair(d, m, wl, KEY_SIGN, math=math, B=B)
        child = np.zeros(wl.n_total, np.uint32)
        score = np.zeros(wl.n_total, np.float32)
        outc = np.zeros(wl.n_total, np.uint8)
        if use_graph:
            bs, bp, bw = (torch.zeros(B, dtype=torch.int32, device="cuda") for _ in range(3))
            sc = torch.zeros(B, dtype=torch.float32, device="cuda")
            ch = torch.zeros(B, dtype=torch.int32, device="cuda")
            oc = torch.zeros(B, dtype=torch.uint8, device="cuda")
            nn = torch.zeros(1, dtype=torch.int32, device="cuda")
            g = eng.graph(B, bs, bp, bw, sc, ch, oc, n=nn)
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            k = sl.stop - sl.start
            par = O.resolve_parents(wl.parent_ref[sl], child)
            if use_graph:
                bs[:k] = _dev(wl.session[sl]); bp[:k] = _dev(par); bw[:k] = _dev(wl.word[sl])
                nn.fill_(k)
                g.launch()
                s_, c_, o_ = sc[:k], ch[:k], oc[:k]
            else:
                s_, c_, o_ = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
            score[sl] = s_.cpu().numpy()
            child[sl] = c_.cpu().numpy().view(np.uint32)
            outc[sl] = o_.cpu().numpy()
        outs.append((score, child, outc, eng.cache_stats()))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][2], outs[1][2])
    assert outs[0][3] == outs[1][3]
    assert outs[0][3]["hidden_hits"] > 0


@pytest.mark.parametrize("math", [MATH_BF16, MATH_FP32])
def test_session_sharded_engines_equal_one_engine(math):
    """SURVEY 8(e) equality test on one GPU: the sessions split over two
    engines (what two ranks of bench.py --gpus 2 hold, parallel.session_range)
    return -- concatenated in session order, as the all-gather assembles them --
    bitwise the scores, handles, outcomes and stats of ONE engine over all
    sessions; large model, 4 staggered streams x 512 queries, sign keys."""
    import torch
    import oracle as O
    from paper_1801_09866_b200.parallel import session_range
    from tests.parity_util import _dev
    d, m = model("large")
    wl = generate_workload(4, 24, 512, d.V, seed=5, dur=(2, 5), eps=0.1).staggered([0, 3, 5, 9])
    parts = [(0, 4)] + [session_range(4, 2, r) for r in range(2)]
    res = {}
    for lo, hi in parts:
        sub = wl.select_sessions(lo, hi)
        eng, _ = pair(d, m, sub, KEY_SIGN, math=math, path=GRU_TILES if math == MATH_BF16 else GRU_GEMV,
                      B=wl.n_per_frame)
        child = np.zeros(sub.n_total, np.uint32)
        score = np.zeros(sub.n_total, np.float32)
        outc = np.zeros(sub.n_total, np.uint8)
        for t in range(sub.frames):
            sl = sub.frame_slice(t)
            if sl.stop == sl.start:
                continue
            par = O.resolve_parents(sub.parent_ref[sl], child)
            s_, c_, o_ = eng.query_batch(_dev(sub.session[sl]), _dev(par), _dev(sub.word[sl]))
            score[sl], child[sl], outc[sl] = s_.cpu().numpy(), c_.cpu().numpy().view(np.uint32), o_.cpu().numpy()
        res[(lo, hi)] = (sub, score, child, outc, eng.cache_stats())
    whole = res[(0, 4)]
    for s in range(4):
        one = [v for (lo, hi), v in res.items() if (lo, hi) != (0, 4) and lo <= s < hi][0]
        a = whole[0].session == s
        b = one[0].session == (s - [lo for (lo, hi) in res if (lo, hi) != (0, 4) and lo <= s < hi][0])
        assert np.array_equal(whole[1][a].view(np.uint32), one[1][b].view(np.uint32))
        assert np.array_equal(whole[2][a], one[2][b]) and np.array_equal(whole[3][a], one[3][b])
    tot = {k: sum(v[4][k] for (lo, hi), v in res.items() if (lo, hi) != (0, 4))
           for k in ("total_queries", "query_hits", "hidden_lookups", "hidden_hits", "gru_computations")}
    assert all(tot[k] == whole[4][k] for k in tot)


@pytest.mark.parametrize("path", [GRU_TILES, GRU_GEMV])
@pytest.mark.parametrize("math", [MATH_FP32, MATH_BF16])
def test_staggered_streams_vs_oracle(math, path):
    """Streams that join at different frames (bench.py's multi workload:
    calls hold only the sessions that have started, session counts vary per
    call) against the oracle, sign keys merging."""
    d, m = model("moderate")
    wl = generate_workload(3, 90, 64, d.V, seed=11, dur=(2, 5), eps=0.1).staggered([0, 7, 19])
    eng, orc = pair(d, m, wl, KEY_SIGN, math=math, path=path)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math])
    assert rep["shit"] > 100, rep
