#!/bin/bash
# Fused GRU kernel diagnostics at a FIXED all-miss size close to the bench step
# (5 sessions x 2,048 queries, cache off: 10,240 GRU rows per step).
# DIAG 0 full, 3 no epilogue work, 5 cycle counters (valid results).
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
RNNLM_NVCC_FLAGS="-DRNNLM_TC_PROF=1" python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1   # cycle counters compiled in
for math in ${MATHS:-bf16 bf16x3}; do for d in ${DIAGS:-0 3 5}; do
  RNNLM_TC_DIAG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --also none \
    --sessions 5 --no-cache --math $math ${DIAG_ARGS:-} > gpurun_out/diag_${math}_d${d}.json 2> gpurun_out/diag_${math}_d${d}.err
  python - gpurun_out/diag_${math}_d${d}.json <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1]); k = d["kernel_ms_per_step"]
    print(f, "gather %.1f us  gru %.1f us  step %.1f us rows/step %.0f" % (k["ms_gru_gather"] * 1e3, k["ms_gru_phase1"] * 1e3, d["ms_per_step"] * 1e3, d["hit_rates"]["gru_rows_per_step"]))
except Exception as e:
    print(f, "failed", e)
PY
  grep 'gru_tc prof' gpurun_out/diag_${math}_d${d}.err | tail -1
done; done
python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1   # back to the default build
