"""The fused small-frame kernel (k_small.cu): a call of at most
RNNLM_GEMV_AUTO_MAX_QUERIES queries on the AUTO path runs as ONE cooperative
kernel.  Checked against the CPU oracle (replay protocol), bitwise against the
multi-kernel GEMV path, under CUDA-graph replay, and on the error paths."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1801_09866_b200 import (GRU_AUTO, GRU_GEMV, INVALID, KEY_OFF, KEY_ROUND, KEY_SIGN, MATH_BF16, MATH_FP32,
                                   MATH_TF32, MATH_TF32X3, MATH_BF16X3, RNNLM)
from synth import generate_workload
from tests.parity_util import _dev, replay_compare
from tests.test_gpu_parity import TOL, forgetful_model, model, pair

pytestmark = pytest.mark.gpu


def _fused_calls(eng):
    t = eng.get_timing(reset=True)
    return t["ms_fused"] > 0


@pytest.mark.parametrize("mode,k", [(KEY_SIGN, 0), (KEY_ROUND, 2), (KEY_OFF, 0)])
def test_tiny_config_fused(mode, k):
    """configs[0] (H = 64, 32 queries x 100 frames, fp32) on the fused kernel."""
    d, m = model("tiny")
    wl = generate_workload(1, 100, 32, d.V, seed=7)
    eng, orc = pair(d, m, wl, mode, k, path=GRU_AUTO)
    eng.set_timing(1)
    rep = replay_compare(eng, orc, wl, tol_score=1e-5, tol_state=1e-5)
    assert _fused_calls(eng)
    assert rep["miss"] > 100


@pytest.mark.parametrize("mode,k", [(KEY_SIGN, 0), (KEY_ROUND, 1), (KEY_ROUND, 2)])
@pytest.mark.parametrize("math", [MATH_BF16, MATH_TF32, MATH_TF32X3, MATH_BF16X3, MATH_FP32])
def test_moderate_fused_lossy(math, mode, k):
    """configs[1] shapes (H = 256, 256 queries/frame) on the lattice stream
    with merging keys, every math mode."""
    d, m = model("moderate")
    wl = generate_workload(1, 200, 256, d.V, seed=7, dur=(2, 6), eps=0.1)
    eng, orc = pair(d, m, wl, mode, k=k, math=math, path=GRU_AUTO)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math])
    assert rep["shit"] >= {(KEY_SIGN, 0): 1500, (KEY_ROUND, 1): 1000, (KEY_ROUND, 2): 300}[(mode, k)], rep


@pytest.mark.parametrize("cell", [1, 2])
@pytest.mark.parametrize("math", [MATH_BF16, MATH_FP32])
def test_fused_cells_multisession(math, cell):
    """LBR / RNN cells, three staggered sessions in one call (sessions join
    at different frames; 64 queries each)."""
    d, m = model("moderate")
    wl = generate_workload(3, 90, 64, d.V, seed=11, dur=(2, 5), eps=0.1).staggered([0, 7, 19])
    eng, orc = pair(d, m, wl, KEY_SIGN, math=math, cell=cell, path=GRU_AUTO)
    rep = replay_compare(eng, orc, wl, tol_score=TOL[math], tol_state=TOL[math])
    assert rep["miss"] > 300


@pytest.mark.parametrize("math", [MATH_BF16, MATH_FP32])
def test_fused_equals_gemv_kernels_bitwise(math):
    """Same decision functions, same per-row GEMV arithmetic: the fused kernel
    and the multi-kernel GEMV path return bitwise the same scores, handles,
    outcomes and states."""
    d, m = model("moderate")
    wl = generate_workload(2, 60, 128, d.V, seed=3, dur=(2, 6), eps=0.1)
    outs = []
    for path in (GRU_AUTO, GRU_GEMV):
        eng, _ = pair(d, m, wl, KEY_SIGN, math=math, path=path)
        child = np.zeros(wl.n_total, np.uint32)
        score = np.zeros(wl.n_total, np.float32)
        outc = np.zeros(wl.n_total, np.uint8)
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            par = O.resolve_parents(wl.parent_ref[sl], child)
            s_, c_, o_ = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
            score[sl], child[sl], outc[sl] = s_.cpu().numpy(), c_.cpu().numpy().view(np.uint32), o_.cpu().numpy()
        states = [eng.read_states(s, child[wl.session == s]).cpu().numpy() for s in range(wl.S)]
        outs.append((score, child, outc, states, eng.cache_stats()))
    a, b = outs
    assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    for x, y in zip(a[3], b[3]):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert a[4] == b[4] and a[4]["hidden_hits"] > 0


def test_fused_graph_replay_with_device_count():
    """The fused kernel captured once (rnnlm_graph_create) and replayed with the
    frame size read on the device, including empty frames (n = 0), equals
    direct calls bitwise."""
    d, m = forgetful_model()
    wl = generate_workload(2, 40, 48, d.V, seed=21, dur=(2, 6), eps=0.3, beam_scale=3).staggered([0, 9])
    B = wl.n_per_frame
    outs = []
    for use_graph in (False, True):
        eng, _ = pair(d, m, wl, KEY_SIGN, B=B, path=GRU_AUTO)
        bufs = [torch.zeros(B, dtype=torch.int32, device="cuda") for _ in range(3)]
        sc = torch.zeros(B, dtype=torch.float32, device="cuda")
        ch = torch.zeros(B, dtype=torch.int32, device="cuda")
        oc = torch.zeros(B, dtype=torch.uint8, device="cuda")
        nn = torch.zeros(1, dtype=torch.int32, device="cuda")
        g = eng.graph(B, *bufs, sc, ch, oc, n=nn) if use_graph else None
        child = np.zeros(wl.n_total, np.uint32)
        score = np.zeros(wl.n_total, np.float32)
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            k = sl.stop - sl.start
            par = O.resolve_parents(wl.parent_ref[sl], child)
            if use_graph:
                for b_, a_ in zip(bufs, (wl.session[sl], par, wl.word[sl])):
                    b_[:k] = _dev(a_)
                nn.fill_(k)
                g.launch()
                if t % 7 == 3:                                 # an empty replay changes nothing
                    nn.fill_(0)
                    g.launch()
                s_, c_ = sc[:k], ch[:k]
            else:
                s_, c_, _ = eng.query_batch(_dev(wl.session[sl]), _dev(par), _dev(wl.word[sl]))
            score[sl], child[sl] = s_.cpu().numpy(), c_.cpu().numpy().view(np.uint32)
        outs.append((score, child, eng.cache_stats()))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1], outs[1][1]) and outs[0][2] == outs[1][2]
    assert outs[0][2]["hidden_hits"] > 0


def test_fused_edge_cases():
    """Invalid queries, same-call duplicates, an unsorted batch (rejected as a
    whole) and capacity exhaustion, on the fused kernel, against the oracle."""
    d, m = model("tiny")
    eng = RNNLM.from_dims(d, m, key_mode=KEY_SIGN, num_sessions=2, max_queries_per_call=512,
                          max_histories_per_session=64, gru_path=GRU_AUTO)
    orc = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_SIGN, 0, 1, 2, 64), m)
    frames = [
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
    # unsorted: every query INVALID, nothing cached; the next call is unaffected
    sc, ch, oc = eng.query_batch(_dev([1, 0]), _dev([0, 0]), _dev([5, 6]))
    assert set(oc.cpu().numpy().tolist()) == {INVALID}
    sess, par, wrd = [0, 0, 1], [1, 2, 1], [11, 12, 13]
    sc, ch, oc = eng.query_batch(_dev(sess), _dev(par), _dev(wrd))
    osc, och, ooc = orc.query_frame(sess, par, wrd)
    assert np.array_equal(oc.cpu().numpy(), ooc) and np.array_equal(ch.cpu().numpy().view(np.uint32), och)
    # capacity: 500 fresh queries on a 64-handle session
    rng = np.random.default_rng(3)
    sess = np.zeros(500)
    par = np.zeros(500)
    wrd = rng.integers(1, d.V, 500)
    sc, ch, oc = eng.query_batch(_dev(sess), _dev(par), _dev(wrd))
    osc, och, ooc = orc.query_frame(sess, par, wrd)
    assert np.array_equal(oc.cpu().numpy(), ooc)
    assert np.array_equal(ch.cpu().numpy().view(np.uint32), och)
    st, ost = eng.cache_stats(), orc.stats()
    for kk in ("total_queries", "query_hits", "hidden_lookups", "hidden_hits", "gru_computations"):
        assert st[kk] == ost[kk]
    assert st["sticky_error"] != 0
