#!/bin/bash
# Timing diagnostics of the fused GRU kernel (results invalid under RNNLM_TC_DIAG):
# DIAG=1 skips the MMAs (TMA loads only), DIAG=2 skips the TMA loads (MMAs only),
# DIAG=3 skips the epilogue work (TMEM drained, counters kept), DIAG=4 = 3 without
# the phase-1 -> phase-2 dependency wait.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
for p in ${PAIRS:-0}; do for d in ${DIAGS:-0 1 2 3 4}; do
  RNNLM_TC_PAIR=$p RNNLM_TC_DIAG=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline ${DIAG_ARGS:-} \
    --timing-level 2 > gpurun_out/diag_p${p}_d${d}.json 2> gpurun_out/diag_p${p}_d${d}.err
done; done
for f in gpurun_out/diag_p*_d*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1]); k = d["kernel_ms_per_step"]
    print(f, "gather %.1f us  gru %.1f us  step %.1f us" % (k["ms_gru_gather"] * 1e3, k["ms_gru_phase1"] * 1e3, d["ms_per_step"] * 1e3))
except Exception as e:
    print(f, "failed", e)
PY
done
