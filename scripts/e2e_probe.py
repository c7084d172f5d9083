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
ref_idx = np.where(wl.parent_ref >= 0, wl.parent_ref, wl.n_total).astype(np.int64)
h_par = torch.empty(n, dtype=torch.int32).pin_memory()
h_score = torch.empty(n, dtype=torch.float32).pin_memory()
h_child = torch.empty(n, dtype=torch.int32).pin_memory()
d_sess = torch.empty(n, dtype=torch.int32, device=dev); d_par = torch.empty_like(d_sess); d_word = torch.empty_like(d_sess)
d_score = torch.empty(n, dtype=torch.float32, device=dev); d_child = torch.empty(n, dtype=torch.int32, device=dev)
child_log = np.zeros(wl.n_total + 1, np.int32)
child_log[:] = 0                      # fault the pages in before the loop
USE_TORCH = len(sys.argv) > 1
log_t = torch.from_numpy(child_log)
ref_t = torch.from_numpy(ref_idx)
par_np, child_np = h_par.numpy(), h_child.numpy()
acc = np.zeros(6)
for t in range(F):
    sl = wl.frame_slice(t)
    t0 = time.perf_counter()
    if USE_TORCH:
        torch.index_select(log_t, 0, ref_t[sl], out=h_par)
    else:
        np.take(child_log, ref_idx[sl], out=par_np)
    t1 = time.perf_counter()
    d_sess.copy_(h_sess_all[sl], non_blocking=True); d_par.copy_(h_par, non_blocking=True); d_word.copy_(h_word_all[sl], non_blocking=True)
    t2 = time.perf_counter()
    eng.query_batch(d_sess, d_par, d_word, score=d_score, child=d_child, want_outcome=False)
    t3 = time.perf_counter()
    h_score.copy_(d_score, non_blocking=True); h_child.copy_(d_child, non_blocking=True)
    t4 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t5 = time.perf_counter()
    child_log[sl] = child_np
    t6 = time.perf_counter()
    if t >= 40:
        acc += np.array([t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5])
acc /= (F - 40)
print("torch" if USE_TORCH else "numpy", torch.get_num_threads(), "per step us: take %.0f  h2d-launch %.0f  query_batch-launch %.0f  d2h-launch %.0f  sync-wait %.0f  log %.0f  total %.0f" % tuple(list(acc * 1e6) + [acc.sum() * 1e6]))
