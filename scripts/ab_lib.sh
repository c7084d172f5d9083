#!/bin/bash
# Same-box A/B of two builds of librnnlm.so (scripts/build_ab.sh puts the
# baseline build at paper_1801_09866_b200/librnnlm_a.so): bench lines
# interleaved, ROUNDS each.  BENCH_ARGS selects the workload.
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
out=gpurun_out/ab_lib.txt; : > $out
for r in $(seq ${ROUNDS:-3}); do
  for v in a b; do
    lib=paper_1801_09866_b200/librnnlm.so; [[ $v == a ]] && lib=paper_1801_09866_b200/librnnlm_a.so
    RNNLM_LIBRARY=$PWD/$lib timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-configs ${BENCH_ARGS:-} > gpurun_out/ab_$v.json 2>/dev/null
    python - $v gpurun_out/ab_$v.json >> $out <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
def one(x):
    k = x["kernel_ms_per_step"]
    return "%s %.1f Mq/s step %.1f us gru %.1f us gather %.1f" % (x.get("dtype", ""), x["value"] / 1e6, x["ms_per_step"] * 1e3,
                                                         k["ms_gru_phase1"] * 1e3, k["ms_gru_gather"] * 1e3)
print(sys.argv[1], one(d), *[" | " + one(d[m]) for m in ("bf16", "tf32x3", "bf16x3") if isinstance(d.get(m), dict)])
PY
  done
done
cat $out
