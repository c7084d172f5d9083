"""Diagnostics: extra CUDA events around resolve_parents / query_batch inside bench.py timed steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, json, time
sys.argv = ["bench.py", "--no-e2e", "--no-cpu-baseline", "--steps", "10", "--warmup", "3", "--timing-level", "0"]
import bench
import torch
# monkeypatch: wrap query_batch to record extra events
import paper_1801_09866_b200 as R
orig_qb = R.RNNLM.query_batch
orig_rp = R.resolve_parents
marks = []
def rp(*a, **k):
    e = torch.cuda.Event(enable_timing=True); e.record(); marks.append(("pre_resolve", e))
    r = orig_rp(*a, **k)
    e = torch.cuda.Event(enable_timing=True); e.record(); marks.append(("post_resolve", e))
    return r
def qb(self, *a, **k):
    r = orig_qb(self, *a, **k)
    e = torch.cuda.Event(enable_timing=True); e.record(); marks.append(("post_qb", e))
    return r
R.resolve_parents = rp
R.RNNLM.query_batch = qb
bench.main()
torch.cuda.synchronize()
# last 10 triples
tr = marks[-30:]
for i in range(0, 30, 3):
    a, b, c = tr[i][1], tr[i + 1][1], tr[i + 2][1]
    print("resolve %.1f us  query_batch %.1f us" % (a.elapsed_time(b) * 1e3, b.elapsed_time(c) * 1e3))
