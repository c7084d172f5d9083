#!/bin/bash
# Timing diagnostics of the fused GRU kernel (results invalid under RNNLM_TC_DIAG):
# DIAG=1 skips the MMAs (TMA loads only), DIAG=2 skips the TMA loads (MMAs only).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
for p in ${PAIRS:-0}; do for d in ${DIAGS:-0 1 2}; do
  RNNLM_TC_PAIR=$p RNNLM_TC_DIAG=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    --timing-level 2 > gpurun_out/diag_p${p}_d${d}.json 2> gpurun_out/diag_p${p}_d${d}.err
done; done
