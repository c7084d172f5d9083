"""Pins of the CPU oracle against values the paper/SPEC and mathematics fix.

Nothing here compares the oracle with a re-typed copy of itself: every
expected value is a worked example (SPEC/PAPER line cited), a hand-derived
closed form (tests/golden/), a library routine in a special case that reduces
to it (torch.nn.GRUCell), or an invariant/brute-force count.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
from synth.model import ModelDims, generate_model, zero_model

pytestmark = pytest.mark.filterwarnings("ignore")


def small_cfg(H, E, V=8, log2=10, N=3, **kw):
    return O.make_config(V, E, H, log2, N, **kw)


# ----------------------------------------------------------------------------- compression
def test_sign_code_spec_S265():
    # mode=sign, h=[0.3,-0.2,0.0] -> bits [1,0,1] (sign(0)=+, reading 5)
    code = O.compress([0.3, -0.2, 0.0], O.KEY_SIGN)
    assert code.tolist() == [0b101]


def test_round2_code_spec_S266_fp32_product():
    # round(2), h=[0.126,-0.005] -> [13,-1].  -0.005f*100 is exactly
    # -0.5 in fp32 (an fp64 product would give -0.49999998 -> 0): reading 4.
    code = O.compress([0.126, -0.005], O.KEY_ROUND, 2).view(np.int8)
    assert code.tolist() == [13, -1]


def test_round_half_away_from_zero_and_widths():
    # 0.125*100 = 12.5 exactly -> 13 (half away; banker's rounding would give 12)
    assert O.compress([0.125, -0.125, 0.0], O.KEY_ROUND, 2).view(np.int8).tolist() == [13, -13, 0]
    # k=1: 0.25*10 = 2.5 -> 3 ; -0.05*10 = -0.5 -> -1
    assert O.compress([0.25, -0.05], O.KEY_ROUND, 1).view(np.int8).tolist() == [3, -1]
    # k=3 uses little-endian int16 (reading 6): 0.5 -> 500, -0.9994 -> -999.4 -> -999
    c = O.compress([0.5, -0.9994], O.KEY_ROUND, 3)
    assert len(c) == 4 and c.view(np.int16).tolist() == [500, -999]
    # k=4: fp32(0.99995) = 0.99994999170; the fp32 product with 10000 rounds to
    # 9999.5 exactly -> 10000 (an fp64 product, 9999.4999, would give 9999)
    assert O.compress([np.float32(0.99995)], O.KEY_ROUND, 4).view(np.int16).tolist() == [10000]


def test_sign_zero_negative_zero_and_bit_order():
    # -0.0 >= 0.0 is true in IEEE: bit 1 (reading 5: never use sign-bit extraction)
    h = np.array([-0.0, 0.5, -1e-30, 0.0, -0.7, 0.1, 0.2, -0.3, 0.9, -0.9], dtype=np.float32)
    code = O.compress(h, O.KEY_SIGN)
    bits = [(int(code[i // 8]) >> (i % 8)) & 1 for i in range(10)]
    assert bits == [1, 1, 0, 1, 0, 1, 1, 0, 1, 0]
    assert len(code) == 2


def test_off_code_is_bit_pattern():
    h = np.array([0.0, -0.0, 0.25], dtype=np.float32)
    c = O.compress(h, O.KEY_OFF)
    assert c.tobytes() == h.tobytes()
    assert O.compress([0.0], O.KEY_OFF).tobytes() != O.compress([-0.0], O.KEY_OFF).tobytes()


def test_round_idempotent_S267():
    rng = np.random.default_rng(0)
    for k, dt in ((1, np.int8), (2, np.int8), (3, np.int16)):
        h = rng.uniform(-1, 1, 1000).astype(np.float32)
        q = O.compress(h, O.KEY_ROUND, k).view(dt).astype(np.float32)
        back = (q / np.float32(10 ** k)).astype(np.float32)
        assert np.array_equal(O.compress(back, O.KEY_ROUND, k), O.compress(h, O.KEY_ROUND, k))


def test_nonfinite_rejected():
    with pytest.raises(ValueError):
        O.compress([np.nan, 0.0], O.KEY_SIGN)


# ----------------------------------------------------------------------------- MaxEnt hash
def test_maxent_spec_S182():
    # M=1000, w=42, ctx=[7]: (42*237967+7+1) mod 1000 = 9,994,622 mod 1000 = 622
    assert O.maxent_indices([7], 42, 3, 1000) == [42, 622]


def test_maxent_empty_context_S183():
    assert O.maxent_indices([], 123457, 4, 1 << 16) == [123457 % 65536]


def test_maxent_context_order_hand():
    # ctx most recent LAST = [3, 9]: order 2 uses 9, order 3 uses 3.
    # idx2 = (5*237967 + 9 + 1) mod 2^16 = 1189845 mod 65536 = 10197
    # idx3 = (10197*237967 + 3 + 1) mod 2^16 = 13567
    assert O.maxent_indices([3, 9], 5, 3, 1 << 16) == [5, 10197, 13567]
    # only the last N-1 words matter
    assert O.maxent_indices([77, 3, 9], 5, 3, 1 << 16) == [5, 10197, 13567]
    # N caps the order
    assert O.maxent_indices([3, 9], 5, 2, 1 << 16) == [5, 10197]


# ----------------------------------------------------------------------------- score
def _score_model(H, V, log2):
    d = ModelDims(V=V, E=1, H=H, maxent_log2=log2, N=2)
    return d, zero_model(d)


def test_nce_score_spec_S173():
    d, m = _score_model(2, 4, 10)
    m["nce_w"][3] = [0.5, -0.3]
    m["nce_b"][3] = 0.1
    cfg = O.make_config(4, 1, 2, 10, 2)
    assert O.score(cfg, m, [1.0, 0.0], [], 3) == pytest.approx(0.6, abs=1e-7)
    # h = 0 -> bias only
    assert O.score(cfg, m, [0.0, 0.0], [], 3) == pytest.approx(0.1, abs=1e-8)


def test_maxent_score_power_of_two_analogue_of_S192():
    # M=1024, w=42, ctx=[7]: idx = [42, (42*237967+8) mod 1024 = 382]
    d, m = _score_model(2, 64, 10)
    m["maxent"][42] = 0.25
    m["maxent"][382] = 0.5
    cfg = O.make_config(64, 1, 2, 10, 2)
    assert O.score(cfg, m, [0.3, 0.7], [7], 42) == 0.75          # NCE part zero
    m["nce_w"][42] = [1.0, 2.0]
    m["nce_b"][42] = 0.125
    # ensemble is additive (reading 13): 0.3 + 1.4 + 0.125 + 0.75
    assert O.score(cfg, m, [0.3, 0.7], [7], 42) == pytest.approx(2.575, abs=1e-6)


def test_score_linear_in_h_S213():
    d = ModelDims(V=50, E=4, H=16, maxent_log2=10, N=3)
    m = generate_model(d, seed=3)
    cfg = O.make_config(50, 4, 16, 10, 3)
    rng = np.random.default_rng(1)
    h1, h2 = rng.uniform(-1, 1, (2, 16)).astype(np.float32)
    a = np.float32(0.5)
    z = np.zeros(16, np.float32)
    base = O.score(cfg, m, z, [1, 2], 7)
    lhs = O.score(cfg, m, (a * h1 + h2).astype(np.float32), [1, 2], 7) - base
    rhs = a * (O.score(cfg, m, h1, [1, 2], 7) - base) + (O.score(cfg, m, h2, [1, 2], 7) - base)
    assert lhs == pytest.approx(rhs, abs=1e-6)


# ----------------------------------------------------------------------------- GRU
def _gru_from_case(c):
    E, H = c["E"], c["H"]
    m = {k: np.array(c[k], dtype=np.float32) for k in
         ("Wz", "Uz", "bz", "Wr", "Ur", "br", "Wh", "Uh", "bh")}
    m.update(emb=np.zeros((2, E), np.float32), nce_w=np.zeros((2, H), np.float32),
             nce_b=np.zeros(2, np.float32), maxent=np.zeros(2, np.float32))
    cfg = O.make_config(2, E, H, 1, 1)
    return cfg, m


def test_gru_hand_cases(golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "gru_hand_cases.json")))["cases"]
    for c in cases:
        cfg, m = _gru_from_case(c)
        out = O.gru(cfg, m, c["x"], c["h"], fp64=True)
        exact_inputs = c["name"] == "spec_S116_scalar"
        tol = 1e-12 if exact_inputs else 1e-7      # ln 3 is not an fp32 number
        np.testing.assert_allclose(out, c["expected"], atol=tol, rtol=0, err_msg=c["name"])
        for wrong in c.get("wrong", {}).values():
            assert np.max(np.abs(out - np.array(wrong))) > 1e-3, c["name"]


def test_gru_zero_weights_halves_state_S115():
    d = ModelDims(V=4, E=8, H=16, maxent_log2=4, N=2)
    m = zero_model(d)
    cfg = O.make_config(4, 8, 16, 4, 2)
    h = np.random.default_rng(2).uniform(-1, 1, 16).astype(np.float32)
    out = O.gru(cfg, m, np.ones(8, np.float32), h)
    assert np.array_equal(out, (np.float32(0.5) * h))


def test_gru_matches_torch_grucell_when_reset_is_one():
    """Special case r == 1 reduces the Chung GRU to a library routine.

    With Wr=Ur=0 and br=40, sigma(40) rounds to 1.0 in fp64, so both
    formulations give tanh(Wh x + Uh h + bh).  torch.nn.GRUCell uses
    h' = (1-z_t) n + z_t h, i.e. z_t = 1 - z = sigma(-(...)): its update-gate
    weights are the negated ones.  This pins W/U orientation (E != H), the
    update-gate orientation, tanh and the biases.
    """
    E, H = 5, 3
    rng = np.random.default_rng(4)
    m = {k: rng.uniform(-1, 1, s).astype(np.float32) for k, s in
         dict(Wz=(H, E), Uz=(H, H), bz=(H,), Wh=(H, E), Uh=(H, H), bh=(H,)).items()}
    m.update(Wr=np.zeros((H, E), np.float32), Ur=np.zeros((H, H), np.float32),
             br=np.full(H, 40.0, np.float32), emb=np.zeros((2, E), np.float32),
             nce_w=np.zeros((2, H), np.float32), nce_b=np.zeros(2, np.float32),
             maxent=np.zeros(2, np.float32))
    x = rng.uniform(-1, 1, E).astype(np.float32)
    h = rng.uniform(-1, 1, H).astype(np.float32)
    cfg = O.make_config(2, E, H, 1, 1)
    ours = O.gru(cfg, m, x, h, fp64=True)

    cell = torch.nn.GRUCell(E, H).double()
    t = lambda a: torch.tensor(a, dtype=torch.float64)
    with torch.no_grad():
        # torch gate order in weight_ih / weight_hh: (r, z, n)
        cell.weight_ih.copy_(torch.cat([t(np.zeros((H, E))), -t(m["Wz"]), t(m["Wh"])]))
        cell.weight_hh.copy_(torch.cat([t(np.zeros((H, H))), -t(m["Uz"]), t(m["Uh"])]))
        cell.bias_ih.copy_(torch.cat([t(np.full(H, 40.0)), -t(m["bz"]), t(m["bh"])]))
        cell.bias_hh.zero_()
        ref = cell(t(x)[None], t(h)[None])[0].numpy()
    np.testing.assert_allclose(ours, ref, atol=1e-13, rtol=0)


def test_gru_zero_history_special_case_S117():
    # h = 0: r*h = 0, so h' = z * tanh(Wh x + bh) with z = sigma(Wz x + bz)
    E, H = 3, 4
    rng = np.random.default_rng(5)
    m = generate_model(ModelDims(V=2, E=E, H=H, maxent_log2=1, N=1), seed=5, scale=1.0,
                       bf16_grid=False)
    cfg = O.make_config(2, E, H, 1, 1)
    x = rng.uniform(-1, 1, E).astype(np.float32)
    out = O.gru(cfg, m, x, np.zeros(H, np.float32), fp64=True)
    X = torch.tensor(x, dtype=torch.float64)
    lin = lambda W, b: torch.nn.functional.linear(X, torch.tensor(W, dtype=torch.float64),
                                                  torch.tensor(b, dtype=torch.float64))
    ref = torch.sigmoid(lin(m["Wz"], m["bz"])) * torch.tanh(lin(m["Wh"], m["bh"]))
    np.testing.assert_allclose(out, ref.numpy(), atol=1e-13, rtol=0)


def test_gru_bounded_state_S129():
    # h' is a convex combination of h in (-1,1) and tanh(.) in (-1,1)
    d = ModelDims(V=2, E=6, H=12, maxent_log2=1, N=1)
    cfg = O.make_config(2, 6, 12, 1, 1)
    rng = np.random.default_rng(6)
    for seed in range(3):
        m = generate_model(d, seed=seed, scale=0.5, bf16_grid=False)
        h = np.zeros(12, np.float32)
        for _ in range(100):
            h64 = O.gru(cfg, m, rng.uniform(-1, 1, 6).astype(np.float32), h, fp64=True)
            assert np.all(np.abs(h64) < 1.0)
            h = h64.astype(np.float32)


# ----------------------------------------------------------------------------- exact log-normaliser (8(f)-2)
def test_log_normalizer_two_equal_words_S206():
    # V=2 with equal scores -> log p = log 0.5 for each word, so
    # log Z = s + ln 2.  Scores set through the bias only (Theta = 0, MaxEnt = 0).
    d, m = _score_model(2, 2, 10)
    m["nce_b"][:] = 0.375
    cfg = O.make_config(2, 1, 2, 10, 2)
    assert O.log_normalizer(cfg, m, [0.3, -0.8], [5]) == pytest.approx(0.375 + math.log(2), abs=1e-12)


def test_log_normalizer_hand_softmax_S208():
    # V=3, combined scores (0, 0, ln 2) -> probabilities (1/4, 1/4, 1/2),
    # i.e. Z = 4.  The third score is ln 2 rounded to fp32 (b_nce is fp32).
    d, m = _score_model(2, 3, 10)
    m["nce_b"][2] = np.float32(math.log(2))
    cfg = O.make_config(3, 1, 2, 10, 2)
    lz = O.log_normalizer(cfg, m, [0.0, 0.0], [])
    assert lz == pytest.approx(math.log(2 + math.exp(float(np.float32(math.log(2))))), abs=1e-12)
    assert lz == pytest.approx(math.log(4), abs=1e-7)
    assert math.exp(float(np.float32(math.log(2))) - lz) == pytest.approx(0.5, abs=1e-7)


def test_log_normalizer_zero_model_is_log_V():
    # every score 0 -> Z = V exactly
    d, m = _score_model(4, 1000, 12)
    cfg = O.make_config(1000, 1, 4, 12, 2)
    assert O.log_normalizer(cfg, m, [0.5, -0.5, 0.25, 1.0], [17]) == pytest.approx(math.log(1000), abs=1e-12)


def test_log_normalizer_single_feature_closed_form():
    # one order-2 MaxEnt weight c at idx_2(ctx=[7], w=42) (M = 1024, N = 2), all
    # else zero: only word 42 hits it (unigram slots of other words are 0 and
    # no other word's order-2 index collides with 382 -- checked), so
    # Z = (V - 1) + e^c.
    d, m = _score_model(2, 64, 10)
    c = 1.5
    m["maxent"][382] = c
    hits = [v for v in range(64) if 382 in O.maxent_indices([7], v, 2, 1024)]
    assert hits == [42]
    cfg = O.make_config(64, 1, 2, 10, 2)
    assert O.log_normalizer(cfg, m, [0.1, 0.2], [7]) == pytest.approx(math.log(63 + math.exp(c)), abs=1e-12)


def test_log_normalizer_sums_to_one_S218():
    # the exact distribution sums to 1 (random models, V <= 1000);
    # per-word scores from the pinned orc_score (fp32-rounded, so ~1e-7 each).
    d = ModelDims(V=300, E=4, H=16, maxent_log2=12, N=4)
    m = generate_model(d, seed=9, scale=1.0)
    cfg = O.make_config(300, 4, 16, 12, 4)
    rng = np.random.default_rng(2)
    h = rng.uniform(-1, 1, 16).astype(np.float32)
    ctx = [11, 250, 3]
    lz = O.log_normalizer(cfg, m, h, ctx)
    p = [math.exp(O.score(cfg, m, h, ctx, v) - lz) for v in range(300)]
    assert sum(p) == pytest.approx(1.0, abs=1e-5)
    assert max(O.score(cfg, m, h, ctx, v) for v in range(300)) <= lz


def test_log_normalizer_shift_invariance():
    # adding c to every NCE bias shifts log Z by exactly c (up to fp32 storage of b + c)
    d = ModelDims(V=64, E=4, H=8, maxent_log2=10, N=3)
    m = generate_model(d, seed=4, scale=1.0)
    cfg = O.make_config(64, 4, 8, 10, 3)
    h = np.linspace(-1, 1, 8).astype(np.float32)
    base = O.log_normalizer(cfg, m, h, [1, 2])
    m2 = dict(m)
    m2["nce_b"] = (m["nce_b"] + np.float32(2.0)).astype(np.float32)
    assert O.log_normalizer(cfg, m2, h, [1, 2]) == pytest.approx(base + 2.0, abs=1e-6)


# ----------------------------------------------------------------------------- cell variant (8(f)-3)
def test_gru_lbr_is_torch_grucell():
    """The linear-before-reset cell IS torch.nn.GRUCell's formulation
    (n = tanh(W_in x + b_in + r . (W_hn h + b_hn))), for arbitrary reset
    gates: with b_hn = 0, b_in = bh and the update gate negated (torch uses
    h' = (1 - z_t) n + z_t h), the library cell is the reference."""
    E, H = 5, 3
    rng = np.random.default_rng(8)
    m = {k: rng.uniform(-1, 1, s).astype(np.float32) for k, s in
         dict(Wz=(H, E), Uz=(H, H), bz=(H,), Wr=(H, E), Ur=(H, H), br=(H,), Wh=(H, E), Uh=(H, H),
              bh=(H,)).items()}
    m.update(emb=np.zeros((2, E), np.float32), nce_w=np.zeros((2, H), np.float32),
             nce_b=np.zeros(2, np.float32), maxent=np.zeros(2, np.float32))
    x = rng.uniform(-1, 1, E).astype(np.float32)
    h = rng.uniform(-1, 1, H).astype(np.float32)
    cfg = O.make_config(2, E, H, 1, 1, cell=O.CELL_GRU_LBR)
    ours = O.gru(cfg, m, x, h, fp64=True)
    cell = torch.nn.GRUCell(E, H).double()
    t = lambda a: torch.tensor(a, dtype=torch.float64)
    with torch.no_grad():
        cell.weight_ih.copy_(torch.cat([t(m["Wr"]), -t(m["Wz"]), t(m["Wh"])]))
        cell.weight_hh.copy_(torch.cat([t(m["Ur"]), -t(m["Uz"]), t(m["Uh"])]))
        cell.bias_ih.copy_(torch.cat([t(m["br"]), -t(m["bz"]), t(m["bh"])]))
        cell.bias_hh.zero_()
        ref = cell(t(x)[None], t(h)[None])[0].numpy()
    np.testing.assert_allclose(ours, ref, atol=1e-13, rtol=0)
    # ... and the default (Chung) cell is NOT that routine when r varies
    chung = O.gru(O.make_config(2, E, H, 1, 1), m, x, h, fp64=True)
    assert np.max(np.abs(chung - ref)) > 1e-3


def test_gru_cells_hand_case_reset_placement():
    """H = 2, E = 1, all weights zero except Uh[0][1] = 1 and br = (0, 40):
    r = (1/2, 1), z = 1/2, x-terms 0.  Unit 0's candidate reads h_1 through Uh:
      Chung: tanh(Uh (r . h))_0 = tanh(r_1 h_1) = tanh(h_1)
      LBR:   tanh(r_0 (Uh h)_0) = tanh(h_1 / 2)
    h'_0 = h_0 / 2 + c_0 / 2; unit 1 has no recurrent input: h'_1 = h_1 / 2."""
    E, H = 1, 2
    m = {k: np.zeros(s, np.float32) for k, s in
         dict(Wz=(H, E), Uz=(H, H), bz=(H,), Wr=(H, E), Ur=(H, H), br=(H,), Wh=(H, E), Uh=(H, H),
              bh=(H,), emb=(2, E), nce_w=(2, H), nce_b=(2,), maxent=(2,)).items()}
    m["Uh"][0, 1] = 1.0
    m["br"][1] = 40.0
    h = np.array([0.25, -0.75], np.float32)
    x = np.array([0.5], np.float32)
    for cell, c0 in ((O.CELL_GRU, math.tanh(-0.75)), (O.CELL_GRU_LBR, math.tanh(-0.375))):
        out = O.gru(O.make_config(2, E, H, 1, 1, cell=cell), m, x, h, fp64=True)
        assert out[0] == pytest.approx(0.125 + 0.5 * c0, abs=1e-15)
        assert out[1] == pytest.approx(-0.375, abs=1e-15)


def test_rnn_cell_hand_case():
    """Vanilla RNN cell (Elman, logistic): H = 2, E = 1, Wh = [[a], [0]],
    Uh = [[0, 1], [0, 0]], bh = (0, b1), every GRU gate weight set to junk
    (must be ignored): h'_0 = sigma(a x + h_1), h'_1 = sigma(b1)."""
    E, H = 1, 2
    rng = np.random.default_rng(3)
    m = {k: rng.uniform(-5, 5, s).astype(np.float32) for k, s in
         dict(Wz=(H, E), Uz=(H, H), bz=(H,), Wr=(H, E), Ur=(H, H), br=(H,)).items()}
    m.update(Wh=np.array([[0.75], [0.0]], np.float32), Uh=np.array([[0.0, 1.0], [0.0, 0.0]], np.float32),
             bh=np.array([0.0, -0.5], np.float32), emb=np.zeros((2, E), np.float32),
             nce_w=np.zeros((2, H), np.float32), nce_b=np.zeros(2, np.float32), maxent=np.zeros(2, np.float32))
    x = np.array([0.5], np.float32)
    h = np.array([0.1, -0.25], np.float32)
    out = O.gru(O.make_config(2, E, H, 1, 1, cell=O.CELL_RNN), m, x, h, fp64=True)
    sig = lambda a: 1.0 / (1.0 + math.exp(-a))
    assert out[0] == pytest.approx(sig(0.375 - 0.25), abs=1e-15)
    assert out[1] == pytest.approx(sig(-0.5), abs=1e-15)


def test_rnn_cell_matches_torch_functional():
    """The Elman layer through torch's library linear + sigmoid (E != H)."""
    E, H = 6, 4
    rng = np.random.default_rng(12)
    m = {k: rng.uniform(-1, 1, s).astype(np.float32) for k, s in
         dict(Wz=(H, E), Uz=(H, H), bz=(H,), Wr=(H, E), Ur=(H, H), br=(H,), Wh=(H, E), Uh=(H, H),
              bh=(H,)).items()}
    m.update(emb=np.zeros((2, E), np.float32), nce_w=np.zeros((2, H), np.float32),
             nce_b=np.zeros(2, np.float32), maxent=np.zeros(2, np.float32))
    x = rng.uniform(-1, 1, E).astype(np.float32)
    h = rng.uniform(-1, 1, H).astype(np.float32)
    ours = O.gru(O.make_config(2, E, H, 1, 1, cell=O.CELL_RNN), m, x, h, fp64=True)
    t = lambda a: torch.tensor(a, dtype=torch.float64)
    ref = torch.sigmoid(torch.nn.functional.linear(t(x), t(m["Wh"]), t(m["bh"])) +
                        torch.nn.functional.linear(t(h), t(m["Uh"]))).numpy()
    np.testing.assert_allclose(ours, ref, atol=1e-13, rtol=0)
