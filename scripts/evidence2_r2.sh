#!/bin/bash
# Round-2 small-frame evidence: per-frame latency of BASELINE configs[0]/[1]
# (direct calls vs CUDA graph; fused / tile / GEMV GRU kernels) and the fused
# small-frame kernel's per-phase durations (RNNLM_SMALL_PROF).
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
: > gpurun_out/latency_r2.jsonl
for cfg in tiny moderate; do for m in bf16 bf16x3 fp32; do
  timeout 600 python scripts/latency_probe.py $cfg $m >> gpurun_out/latency_r2.jsonl 2>> gpurun_out/latency.err
done; done
RNNLM_SMALL_PROF=1 timeout 600 python scripts/latency_probe.py moderate bf16 auto 2>&1 | grep 'k_small prof' | tail -200 > gpurun_out/small_phases_r2.txt
RNNLM_SMALL_PROF=1 timeout 600 python scripts/latency_probe.py tiny fp32 auto 2>&1 | grep 'k_small prof' | tail -60 >> gpurun_out/small_phases_r2.txt
wc -l gpurun_out/latency_r2.jsonl gpurun_out/small_phases_r2.txt
