"""cuBLAS reference point for the fused GRU kernel: the same two contractions
as plain library GEMMs (no gates, no gather, no state update, no codes) at the
bench step's GRU row counts.  Phase 1: [Q, E+H] x [E+H, 2H] (z, r); phase 2:
[Q, E+H] x [E+H, H] (candidate).  bf16 operands, fp32 accumulation (torch
matmul, bf16 output); CUDA events, best of 20 after warm-up.  Prints JSON."""
import json
import sys

import torch

E = H = 1024
out = []
for Q in [int(x) for x in (sys.argv[1:] or ["9984", "10240", "16384", "32768"])]:
    a = torch.randn(Q, E + H, device="cuda", dtype=torch.bfloat16)
    w1 = torch.randn(E + H, 2 * H, device="cuda", dtype=torch.bfloat16)
    w2 = torch.randn(E + H, H, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        torch.matmul(a, w1); torch.matmul(a, w2)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, w1)
        torch.matmul(a, w2)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    fl = 2.0 * Q * (E + H) * 3 * H
    out.append({"rows": Q, "cublas_two_gemms_us": best * 1e3, "tflops": fl / (best * 1e-3) / 1e12})
print(json.dumps({"what": "cuBLAS bf16 GEMMs of the GRU contraction shapes (no epilogue work)", "results": out}))
