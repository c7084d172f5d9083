"""Is the single-stream frame loop of bench.py host-bound?  For the tiny and
moderate configs: the host time to enqueue the timed frames (no sync) and the
device interval, for (A) bench.py's frame_loop calls (torch slicing + the
Python wrappers per frame) and (B) the same C ABI calls with every pointer
precomputed (what a C/C++ decoder pays per frame).

    python scripts/host_rate_probe.py > gpurun_out/host_rate.jsonl
"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1801_09866_b200 as R  # noqa: E402
from paper_1801_09866_b200 import _lib  # noqa: E402
from synth import generate_model  # noqa: E402


def run(name, math, key, lean):
    dev = torch.device("cuda:0")
    d, wl = bench.single_stream(name)
    m = generate_model(d, seed=1234)
    mode, k = bench.key_mode(key)
    eng = R.RNNLM.from_dims(d, m, key_mode=mode, round_digits=k, math=bench.math_id(math), num_sessions=1,
                            max_queries_per_call=wl.n_per_frame, max_histories_per_session=wl.max_histories_hint())
    n, F = wl.n_per_frame, wl.frames
    t_lo = min(40, F // 2)
    d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
    d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
    d_ref = torch.as_tensor(wl.parent_ref, device=dev)
    d_child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    d_score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
    par = torch.zeros(n, dtype=torch.int32, device=dev)
    lib = _lib.load()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    h = eng._h
    sl = [wl.frame_slice(t) for t in range(F)]
    pre = [(sl[t].stop - sl[t].start, ctypes.c_void_p(d_ref[sl[t]].data_ptr()), ctypes.c_void_p(d_sess[sl[t]].data_ptr()),
            ctypes.c_void_p(d_word[sl[t]].data_ptr()), ctypes.c_void_p(d_score[sl[t]].data_ptr()),
            ctypes.c_void_p(d_child[sl[t]].data_ptr())) for t in range(F)]
    p_par, p_child_all = ctypes.c_void_p(par.data_ptr()), ctypes.c_void_p(d_child.data_ptr())

    def frame(t):
        if lean:
            nn, pr, ps, pw, psc, pch = pre[t]
            lib.rnnlm_resolve_parents(nn, pr, p_child_all, p_par, st)
            lib.rnnlm_query_batch(h, nn, ps, p_par, pw, psc, pch, None, st)
        else:
            s_ = sl[t]
            R.resolve_parents(d_ref[s_], d_child, par)
            eng.query_batch(d_sess[s_], par, d_word[s_], score=d_score[s_], child=d_child[s_], want_outcome=False)

    for t in range(t_lo):
        frame(t)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    h0 = time.perf_counter()
    for t in range(t_lo, F):
        frame(t)
    h1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    nf = F - t_lo
    out = {"config": name, "math": math, "key": key, "calls": "lean ctypes (precomputed pointers)" if lean else "bench frame_loop",
           "host_us_per_frame": 1e6 * (h1 - h0) / nf, "device_us_per_frame": 1e3 * a.elapsed_time(b) / nf}
    eng.close()
    return out


if __name__ == "__main__":
    for name, math, key in (("tiny", "fp32", "sign"), ("moderate", "bf16", "sign"), ("moderate", "bf16x3", "sign")):
        for lean in (False, True):
            print(json.dumps(run(name, math, key, lean)), flush=True)
