#!/bin/bash
# Epilogue knock-outs (librnnlm_ko<k>.so built with -DEPI_KO=k; results invalid,
# timing only): fused GRU kernel time at a fixed all-miss size (10,240 rows).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
out=gpurun_out/ab_epi_ko.txt; : > $out
for r in 1 2; do
for lib in librnnlm.so ${KO_LIBS:-librnnlm_ko16.so librnnlm_ko1.so librnnlm_ko2.so}; do
  for math in bf16 bf16x3; do
    RNNLM_LIBRARY=$PWD/paper_1801_09866_b200/$lib timeout 120 python bench.py --steps 10 --warmup 3 \
      --no-e2e --no-cpu-baseline --no-configs --also none --sessions 5 --no-cache --math $math > gpurun_out/ko.json 2>/dev/null
    python - $lib $math gpurun_out/ko.json >> $out <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1]); k = d["kernel_ms_per_step"]
    print(sys.argv[1], sys.argv[2], "gru %.1f us" % (k["ms_gru_phase1"] * 1e3))
except Exception as e:
    print(sys.argv[1:3], "failed", e)
PY
  done
done
done
cat $out
