#!/bin/bash
# Epilogue knock-outs (builds librnnlm_ko<k>.so with -DEPI_KO=k; results invalid,
# timing only): kernel time of the fused GRU at a fixed all-miss size, full
# kernel (diag 0) and epilogue alone (diag 6).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
out=gpurun_out/ab_epi_ko.txt; : > $out
for lib in librnnlm.so librnnlm_ko1.so librnnlm_ko2.so librnnlm_ko3.so librnnlm_ko8.so; do
  for math in bf16 bf16x3; do for d in 0 6; do
    RNNLM_LIBRARY=$PWD/paper_1801_09866_b200/$lib RNNLM_TC_DIAG=$d timeout 300 python bench.py --steps 10 --warmup 3 \
      --no-e2e --no-cpu-baseline --no-configs --also none --sessions 5 --no-cache --math $math > gpurun_out/ko.json 2>/dev/null
    python - $lib $math $d gpurun_out/ko.json >> $out <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[4]).read().strip().splitlines()[-1]); k = d["kernel_ms_per_step"]
    print(sys.argv[1], sys.argv[2], "diag", sys.argv[3], "gru %.1f us" % (k["ms_gru_phase1"] * 1e3))
except Exception as e:
    print(sys.argv[1:4], "failed", e)
PY
  done; done
done
cat $out
