#!/usr/bin/env python
"""BASELINE.json configs[3] (history-compression sweep) and SURVEY 8(f)-1
(per-query vs frame-batched ablation, the paper's Table 2 on B200).

    python scripts/sweep.py --what sweep    [--sessions 16 --frames 120]
    python scripts/sweep.py --what ablation [--config moderate --frames 40]

Writes one JSON object per line to stdout.

Sweep: the large model (V=200k, H=E=1024, 2^27 4-gram), modes off / round:3 /
round:2 / round:1 / sign on the same seeded stream.  Reported per mode: the
LM-query and hidden-cache hit rates, unique GRU computations and the
redundancy rate vs mode off (Table 1's formula), queries/s of the
BF16 tensor-core step, and the score deviation of the lossy mode from exact
evaluation (mode off on the FP32 path, which tests/ pin to the CPU oracle
within 1e-5).  QHIT decisions are exact in every mode, so the same queries
get the same handles and are compared one to one.

Ablation: the same stream once with one rnnlm_query_batch call per decoder
frame and once with one call per query ("more than a hundred
thousand data exchanges"), results checked bitwise equal.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1801_09866_b200 as R  # noqa: E402
from paper_1801_09866_b200 import redundancy_rate  # noqa: E402
from synth import CONFIGS, generate_model, generate_workload, model_dims  # noqa: E402


def run(dims, model, wl, key, math, warm=5, timed_from=None):
    mode, k = R.KEY_MODES[key]
    eng = R.RNNLM.from_dims(dims, model, key_mode=mode, round_digits=k, math=math,
                            num_sessions=wl.S, max_queries_per_call=wl.n_per_frame,
                            max_histories_per_session=wl.max_histories_hint())
    dev = torch.device("cuda")
    d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
    d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
    d_ref = torch.as_tensor(wl.parent_ref, device=dev)
    d_child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    d_score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
    d_par = torch.zeros(wl.n_per_frame, dtype=torch.int32, device=dev)
    t0 = timed_from if timed_from is not None else warm
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for t in range(wl.frames):
        if t == t0:
            torch.cuda.synchronize()
            ev[0].record()
        sl = wl.frame_slice(t)
        R.resolve_parents(d_ref[sl], d_child, d_par)
        eng.query_batch(d_sess[sl], d_par, d_word[sl], score=d_score[sl], child=d_child[sl],
                        want_outcome=False)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    st = eng.cache_stats()
    qps = (wl.frames - t0) * wl.n_per_frame / (ms / 1e3)
    return st, qps, d_score.cpu().numpy(), d_child.cpu().numpy().view(np.uint32)


MATHS = {"bf16": R.MATH_BF16, "bf16x3": R.MATH_BF16X3, "tf32x3": R.MATH_TF32X3, "tf32": R.MATH_TF32,
         "fp32": R.MATH_FP32}


def sweep(a):
    cfg = a.config
    dims = model_dims(cfg)
    model = generate_model(dims, seed=1234)
    wl = generate_workload(a.sessions, a.frames, CONFIGS[cfg]["B_s"], dims.V, seed=7)
    ref_st, _, ref_sc, ref_ch = run(dims, model, wl, "off", R.MATH_FP32)
    base = None
    for key in ("off", "round:3", "round:2", "round:1", "sign"):
        st, qps, sc, ch = run(dims, model, wl, key, MATHS[a.math])
        assert np.array_equal(ch, ref_ch), "QHIT decisions / handles differ across modes"
        dev = np.abs(sc.astype(np.float64) - ref_sc.astype(np.float64))
        if base is None:
            base = st["gru_computations"]
        print(json.dumps({
            "sweep": "compression", "config": cfg, "mode": key, "math": a.math, "sessions": wl.S,
            "frames": wl.frames, "queries": st["total_queries"],
            "query_cache_hit_rate": st["query_hits"] / st["total_queries"],
            "hidden_cache_hit_rate": st["hidden_hits"] / max(1, st["hidden_lookups"]),
            "unique_gru": st["gru_computations"],
            "redundancy_rate_pct": redundancy_rate(base, st["gru_computations"]),
            "queries_per_s": qps,
            "score_dev_vs_exact": {"max": float(dev.max()), "mean": float(dev.mean())},
            "reference": "FP32 path, mode off (pinned to the CPU oracle within 1e-5)"}),
            flush=True)


def ablation(a):
    cfg = CONFIGS[a.config]
    dims = model_dims(a.config)
    model = generate_model(dims, seed=1234)
    wl = generate_workload(1, a.frames, cfg["B_s"], dims.V, seed=7)
    math = MATHS[a.math]
    st, qps_frame, sc_f, ch_f = run(dims, model, wl, "off", math, warm=0)
    # one call per query
    eng = R.RNNLM.from_dims(dims, model, key_mode=R.KEY_OFF, math=math, num_sessions=1,
                            max_queries_per_call=wl.n_per_frame,
                            max_histories_per_session=wl.max_histories_hint())
    dev = torch.device("cuda")
    d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
    d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
    d_ref = torch.as_tensor(wl.parent_ref, device=dev)
    d_child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    d_score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
    d_par = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(wl.frames):
        sl = wl.frame_slice(t)
        R.resolve_parents(d_ref[sl], d_child, d_par[sl])
        for i in range(sl.start, sl.stop):
            eng.query_batch(d_sess[i:i + 1], d_par[i:i + 1], d_word[i:i + 1], score=d_score[i:i + 1],
                            child=d_child[i:i + 1], want_outcome=False)
    e1.record()
    torch.cuda.synchronize()
    qps_query = wl.n_total / (e0.elapsed_time(e1) / 1e3)
    same = (np.array_equal(d_child.cpu().numpy().view(np.uint32), ch_f) and
            np.array_equal(d_score.cpu().numpy().view(np.uint32), sc_f.view(np.uint32)))
    print(json.dumps({"ablation": "per-query vs per-frame", "config": a.config, "math": a.math,
                      "frames": wl.frames, "queries": wl.n_total,
                      "calls_per_query_mode": wl.n_total, "calls_per_frame_mode": wl.frames,
                      "queries_per_s_per_frame": qps_frame, "queries_per_s_per_query": qps_query,
                      "speedup_frame_batching": qps_frame / qps_query,
                      "results_bitwise_equal": bool(same)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="sweep", choices=["sweep", "ablation"])
    ap.add_argument("--sessions", type=int, default=16)
    ap.add_argument("--frames", type=int, default=120)
    ap.add_argument("--config", default=None, help="sweep: large (default); ablation: moderate")
    ap.add_argument("--math", default="bf16")
    a = ap.parse_args()
    if a.config is None:
        a.config = "large" if a.what == "sweep" else "moderate"
    (sweep if a.what == "sweep" else ablation)(a)


if __name__ == "__main__":
    main()
