"""GPU parity of the exact log-normaliser (rnnlm_log_normalizer)
against the CPU oracle's fp64 log sum_v exp(score_v).

Protocol: a seeded workload is replayed through both sides with
tests.parity_util.replay_compare, which overwrites the oracle's new states with
the GPU's, so afterwards every stored history (state + context) is identical
on both sides and log Z is compared on the same inputs.  Tolerance: 1e-3
absolute (the tensor-core tolerance of the north_star); the state enters the
contraction as two bf16 halves, so the observed error is far below it.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1801_09866_b200 import KEY_SIGN, MATH_BF16, MATH_FP32, MATH_TF32, RNNLM
from synth import generate_model, generate_workload, model_dims
from synth.model import ModelDims
from tests.parity_util import _dev, replay_compare

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _replayed(d, m, wl, math):
    cap = wl.max_histories_hint()
    eng = RNNLM.from_dims(d, m, key_mode=KEY_SIGN, math=math, num_sessions=wl.S,
                          max_queries_per_call=max(wl.n_per_frame, 512), max_histories_per_session=cap)
    orc = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_SIGN, 0, 1, wl.S, cap), m)
    replay_compare(eng, orc, wl, tol_score=1e-3, tol_state=1e-3)
    return eng, orc


def _check(eng, orc, pairs):
    sess = np.array([p[0] for p in pairs], np.uint32)
    hist = np.array([p[1] for p in pairs], np.uint32)
    got = eng.log_normalizer(_dev(sess), _dev(hist)).cpu().numpy().astype(np.float64)
    want = np.empty(len(pairs))
    for s in np.unique(sess):
        m = sess == s
        want[m] = orc.log_normalizer(int(s), hist[m]) if s < orc.cfg.num_sessions else np.nan
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    err = float(np.max(np.abs(got[ok] - want[ok]))) if ok.any() else 0.0
    assert err <= TOL, err
    return err


@pytest.mark.parametrize("math,H", [(MATH_FP32, 64), (MATH_BF16, 256), (MATH_TF32, 256)])
def test_small_vocab_all_handles_and_invalid(math, H):
    """Every history of two sessions (contexts of every length, the root) plus
    handles that do not exist (NaN); ragged last M-tile.  H = 64 is the tiny
    config (FP32 engine); the tensor-core GRU paths need H % 256 == 0."""
    d = ModelDims(V=1000, E=H, H=H, maxent_log2=16, N=3)
    m = generate_model(d, seed=1234)
    wl = generate_workload(2, 12, 32, d.V, seed=7)
    eng, orc = _replayed(d, m, wl, math)
    nh = [orc.num_handles(s)[0] for s in range(2)]
    pairs = [(s, h) for s in range(2) for h in range(nh[s])]
    pairs += [(0, nh[0]), (1, nh[1] + 5), (7, 0)]          # unknown handle, unknown session
    err = _check(eng, orc, pairs)
    assert err < 1e-4, err


def test_moderate_two_tiles_ragged():
    """Moderate model (V = 100k, H = 256, 4-gram MaxEnt 2^22): 200 histories =
    one full and one ragged 128-row tile, 391 word tiles (last ragged)."""
    d, m = model_dims("moderate"), None
    m = generate_model(d, seed=1234)
    wl = generate_workload(1, 6, 64, d.V, seed=11)
    eng, orc = _replayed(d, m, wl, MATH_BF16)
    nh = orc.num_handles(0)[0]
    pairs = [(0, h) for h in range(min(nh, 200))]
    _check(eng, orc, pairs)


def test_large_sampled_rows_of_full_batch():
    """Large model (V = 200k, H = 1024, MaxEnt 2^27): log Z of a 512-history
    batch computed in one call; 6 rows spread over the M-tiles checked
    against the oracle (the fp64 oracle takes ~0.3 s per history here)."""
    d = model_dims("large")
    m = generate_model(d, seed=1234)
    wl = generate_workload(1, 3, 256, d.V, seed=5)
    eng, orc = _replayed(d, m, wl, MATH_BF16)
    nh = orc.num_handles(0)[0]
    hist = np.arange(512, dtype=np.uint32) % nh
    got = eng.log_normalizer(_dev(np.zeros(512, np.uint32)), _dev(hist)).cpu().numpy()
    rows = [0, 127, 128, 300, 384, 511]
    want = orc.log_normalizer(0, hist[rows])
    assert np.max(np.abs(got[rows] - want)) <= TOL
    # the same history anywhere in the batch gives the same value (row independence)
    same = hist == hist[300]
    assert np.all(got[same] == got[300])


def test_log_probabilities_sum_to_one_on_gpu():
    """exp(score - log Z) over the whole vocabulary sums to 1: the scores of
    every word from rnnlm_query_batch against one history (the root of a
    fresh utterance, then a child of it) and that history's log Z."""
    d = ModelDims(V=1000, E=64, H=64, maxent_log2=16, N=3)
    m = generate_model(d, seed=1234, scale=1.0)
    eng = RNNLM.from_dims(d, m, key_mode=KEY_SIGN, math=MATH_FP32, num_sessions=1,
                          max_queries_per_call=d.V, max_histories_per_session=3 * d.V)
    zeros = _dev(np.zeros(d.V, np.uint32))
    words = _dev(np.arange(d.V, dtype=np.uint32))
    lz0 = float(eng.log_normalizer(zeros[:1], zeros[:1]).cpu()[0])
    sc, ch, _ = eng.query_batch(zeros, zeros, words)
    p0 = np.exp(sc.cpu().numpy().astype(np.float64) - lz0)
    assert abs(p0.sum() - 1.0) < 1e-5
    child = int(ch.cpu()[37])
    lz1 = float(eng.log_normalizer(zeros[:1], _dev([child])).cpu()[0])
    sc1, _, _ = eng.query_batch(zeros, _dev(np.full(d.V, child, np.uint32)), words)
    p1 = np.exp(sc1.cpu().numpy().astype(np.float64) - lz1)
    assert abs(p1.sum() - 1.0) < 1e-5
    assert abs(lz1 - lz0) > 1e-3          # a different history, a different normaliser


@pytest.mark.parametrize("math", [MATH_FP32, MATH_TF32, MATH_BF16])
def test_off_grid_output_weights(math):
    """Output rows NOT on the bf16 grid (U(-0.1, 0.1) fp32, SPEC S:62 scale):
    the normaliser splits Theta into bf16 hi + lo parts and adds the
    h_hi . Theta_lo product, so log Z stays far inside 1e-3 (a single bf16
    rounding of Theta alone gives ~1e-3 at H = 256).  On the BF16 engine the
    scores themselves round Theta (nce_w is kept fp32 when not bf16-exact)."""
    d = ModelDims(V=3000, E=256, H=256, maxent_log2=16, N=3)
    m = generate_model(d, seed=5, scale=0.1, bf16_grid=False)
    wl = generate_workload(1, 10, 64, d.V, seed=11)
    cap = wl.max_histories_hint()
    eng = RNNLM.from_dims(d, m, key_mode=KEY_SIGN, math=math, num_sessions=1,
                          max_queries_per_call=512, max_histories_per_session=cap)
    orc = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_SIGN, 0, 1, 1, cap), m)
    replay_compare(eng, orc, wl, tol_score=1e-2, tol_state=1e-2)
    nh = orc.num_handles(0)[0]
    err = _check(eng, orc, [(0, h) for h in range(nh)])
    assert err < 1e-4, err
