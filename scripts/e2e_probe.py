"""Diagnostics: host-side cost breakdown of bench.py's e2e loop (not a bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1801_09866_b200 as R
from synth import generate_model, generate_workload, model_dims

d = model_dims("large")
m = generate_model(d, seed=1234)
S, B_s, F = 64, 2048, 60
wl = generate_workload(S, F, B_s, d.V, seed=7)
n = wl.n_per_frame
eng = R.RNNLM.from_dims(d, m, key_mode=R.KEY_SIGN, math=R.MATH_BF16, num_sessions=S,
                        max_queries_per_call=n, max_histories_per_session=wl.max_histories_hint())
dev = torch.device("cuda", 0)
h_sess_all = torch.from_numpy(wl.session.view(np.int32).copy()).pin_memory()
h_word_all = torch.from_numpy(wl.word.view(np.int32).copy()).pin_memory()
h_ref_all = torch.from_numpy(np.ascontiguousarray(wl.parent_ref, dtype=np.int64)).pin_memory()
h_score = torch.empty(n, dtype=torch.float32).pin_memory()
h_child = torch.empty(n, dtype=torch.int32).pin_memory()
d_sess = torch.empty(n, dtype=torch.int32, device=dev); d_word = torch.empty_like(d_sess)
d_ref = torch.empty(n, dtype=torch.int64, device=dev); d_par = torch.empty(n, dtype=torch.int32, device=dev)
d_score = torch.empty(n, dtype=torch.float32, device=dev)
d_child_log = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
acc = np.zeros(5)
for t in range(F):
    sl = wl.frame_slice(t)
    t0 = time.perf_counter()
    d_sess.copy_(h_sess_all[sl], non_blocking=True); d_ref.copy_(h_ref_all[sl], non_blocking=True); d_word.copy_(h_word_all[sl], non_blocking=True)
    t1 = time.perf_counter()
    R.resolve_parents(d_ref, d_child_log, d_par)
    eng.query_batch(d_sess, d_par, d_word, score=d_score, child=d_child_log[sl], want_outcome=False)
    t2 = time.perf_counter()
    h_score.copy_(d_score, non_blocking=True); h_child.copy_(d_child_log[sl], non_blocking=True)
    t3 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t4 = time.perf_counter()
    if t >= 40:
        acc += np.array([t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0])
acc /= (F - 40)
print("per step us: h2d %.0f  resolve+query_batch %.0f  d2h %.0f  sync-wait %.0f  total %.0f" % tuple(acc * 1e6))
