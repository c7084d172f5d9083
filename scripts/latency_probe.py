"""Per-frame latency of small single-session frames (BASELINE configs[0]/[1]):
direct rnnlm_query_batch calls vs a replayed CUDA graph, tile vs GEMV GRU
kernels.  Prints one JSON line per variant (diagnostics; bench.py reports the
numbers that count)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1801_09866_b200 as R  # noqa: E402
from synth import CONFIGS, generate_model, generate_workload, model_dims  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "moderate"
math = {"bf16": R.MATH_BF16, "fp32": R.MATH_FP32, "tf32x3": R.MATH_TF32X3, "bf16x3": R.MATH_BF16X3}[sys.argv[2] if len(sys.argv) > 2 else "bf16"]
c = CONFIGS[cfg]
d = model_dims(cfg)
m = generate_model(d, seed=1234)
wl = generate_workload(1, c["frames"], c["B_s"], d.V, seed=7)
n = wl.n_per_frame
dev = torch.device("cuda", 0)
d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
d_ref = torch.as_tensor(wl.parent_ref, device=dev)
paths = ([R.GRU_AUTO, R.GRU_TILES, R.GRU_GEMV] if d.H % 128 == 0 or math == R.MATH_FP32
         else [R.GRU_AUTO, R.GRU_GEMV])
if len(sys.argv) > 3:
    paths = [{"auto": R.GRU_AUTO, "tiles": R.GRU_TILES, "gemv": R.GRU_GEMV}[sys.argv[3]]]
for path in paths:
    for use_graph in (False, True):
        eng = R.RNNLM.from_dims(d, m, key_mode=R.KEY_SIGN, math=math, num_sessions=1, max_queries_per_call=n,
                                max_histories_per_session=wl.max_histories_hint(), gru_path=path)
        d_child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
        d_score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
        par = torch.zeros(n, dtype=torch.int32, device=dev)
        bs, bw = torch.zeros(n, dtype=torch.int32, device=dev), torch.zeros(n, dtype=torch.int32, device=dev)
        sc, ch = torch.zeros(n, dtype=torch.float32, device=dev), torch.zeros(n, dtype=torch.int32, device=dev)
        g = eng.graph(n, bs, par, bw, sc, ch) if use_graph else None

        def frame(t):
            sl = wl.frame_slice(t)
            R.resolve_parents(d_ref[sl], d_child, par)
            if g is not None:
                bs.copy_(d_sess[sl]); bw.copy_(d_word[sl])
                g.launch()
                d_child[sl].copy_(ch); d_score[sl].copy_(sc)
            else:
                eng.query_batch(d_sess[sl], par, d_word[sl], score=d_score[sl], child=d_child[sl], want_outcome=False)
        for t in range(40):
            frame(t)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        for t in range(40, wl.frames):
            frame(t)
        b.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        F = wl.frames - 40
        print(json.dumps({"config": cfg, "math": sys.argv[2] if len(sys.argv) > 2 else "bf16",
                          "path": {R.GRU_AUTO: "auto (fused when n <= 512)", R.GRU_TILES: "tiles", R.GRU_GEMV: "gemv"}[path], "graph": use_graph,
                          "us_per_frame_gpu": 1e3 * a.elapsed_time(b) / F, "us_per_frame_wall": 1e6 * wall / F,
                          "q_per_s": n * F / wall, "stats": eng.cache_stats()}), flush=True)
        del g, eng
