"""Throughput of the exact log-normaliser (rnnlm_log_normalizer)
on the large model (V = 200k, H = 1024, 4-gram MaxEnt 2^27): log Z of
`--histories` distinct stored histories per call (the 2,048 queries/frame of
BASELINE configs[2]), device-timed with CUDA events; one JSON line.

Roofline of the dominant kernel (k_norm_tc): its algorithmic traffic is the
MaxEnt gathers, (K - 1) random 4-byte reads = 32-byte sectors per (history,
word) (K = 4 orders; order 1 is a per-word bias), plus one pass over the bf16
output rows per 128-history tile; the contraction (two bf16 MMAs per element
pair) is reported beside it.  Inputs: synthetic, seeded (synth/).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--histories", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--math", default="bf16", choices=["bf16", "tf32", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_1801_09866_b200 as R
    from synth import generate_model, generate_workload, model_dims

    d = model_dims("large")
    m = generate_model(d, seed=1234)
    n = args.histories
    # distinct histories: one utterance, cache off, 2 frames of n/2 queries
    # each -> every query makes a new history (depth 1 and 2)
    wl = generate_workload(1, 2, n // 2, d.V, seed=5)
    math = {"bf16": R.MATH_BF16, "tf32": R.MATH_TF32, "fp32": R.MATH_FP32}[args.math]
    eng = R.RNNLM.from_dims(d, m, key_mode=R.KEY_SIGN, math=math, cache_enabled=False, num_sessions=1,
                            max_queries_per_call=n, max_histories_per_session=n + 2)
    dev = torch.device("cuda", 0)
    child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    ref = torch.as_tensor(wl.parent_ref, device=dev)
    par = torch.zeros(wl.n_per_frame, dtype=torch.int32, device=dev)
    for t in range(wl.frames):
        sl = wl.frame_slice(t)
        R.resolve_parents(ref[sl], child, par)
        s_ = torch.as_tensor(wl.session[sl].view(np.int32), device=dev)
        w_ = torch.as_tensor(wl.word[sl].view(np.int32), device=dev)
        eng.query_batch(s_, par, w_, score=torch.empty(wl.n_per_frame, device=dev), child=child[sl],
                        want_outcome=False)
    torch.cuda.synchronize()
    hist = torch.arange(1, n + 1, dtype=torch.int32, device=dev)       # handles 1..n (0 = root)
    sess = torch.zeros(n, dtype=torch.int32, device=dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        eng.log_normalizer(sess, hist, out=out)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in evs:
        a.record()
        eng.log_normalizer(sess, hist, out=out)
        b.record()
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    assert torch.isfinite(out).all()
    K = d.N
    sectors = n * d.V * (K - 1) * 32.0
    theta = -(-n // 128) * d.V * d.H * 2.0
    flops = 2.0 * 2.0 * n * d.V * d.H
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6458.1)
    gbs = (sectors + theta) / (ms * 1e-3) / 1e9
    line = {
        "metric": "exact log-normalisers/sec (large model, V=200k, 4-gram MaxEnt)", "value": n / (ms * 1e-3),
        "unit": "histories/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "dtype": "bf16x2", "data": "synthetic",
        "config": {"workload": "normalizer", "histories_per_call": n, "V": d.V, "H": d.H,
                   "maxent": f"2^{d.maxent_log2} {d.N}-gram", "engine_math": args.math,
                   "l2": "inputs (1.6 GB of gathers + 6.5 GB of output rows per call) exceed L2"},
        "roofline": {"kernel": "k_norm_tc (contraction + MaxEnt gathers + online log-sum-exp)", "bound": "hbm",
                     "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                     "algorithmic": f"{n} x {d.V} x {K - 1} random 32-B MaxEnt sectors + {-(-n // 128)} passes "
                                    f"over the bf16 output rows",
                     "traffic": None, "contraction_tflops": flops / (ms * 1e-3) / 1e12},
    }
    if not args.no_cpu_baseline:
        import oracle as O
        orc = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_OFF, 0, 0, 1, n + 2), m)
        st = eng.read_states(0, np.arange(1, 3, dtype=np.uint32)).cpu().numpy()
        t0 = time.perf_counter()
        cfg = O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N)
        for i in range(2):
            O.log_normalizer(cfg, m, st[i], [int(wl.word[i])])
        secs = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": 2 / secs, "unit": "histories/s", "cores": 1, "kind": "oracle",
                                "sample": f"2 histories ({secs:.1f} s)"}
        del orc
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
