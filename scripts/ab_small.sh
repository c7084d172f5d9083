#!/bin/bash
# A/B of the fused small-frame kernel: CTA count (RNNLM_SMALL_GRID) and the
# barrier spin's nanosleep (build knob RNNLM_SMALL_SLEEP); moderate bf16.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
for sl in 0 32; do
  RNNLM_NVCC_FLAGS="-DRNNLM_SMALL_SLEEP=$sl" python -c "from paper_1801_09866_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  for g in 8 16 32 64 148; do
    echo "sleep=$sl grid=$g $(RNNLM_SMALL_GRID=$g timeout 300 python scripts/latency_probe.py moderate bf16 auto 2>&1 | head -1)"
  done
done > gpurun_out/ab_small.txt
python -c "from paper_1801_09866_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
