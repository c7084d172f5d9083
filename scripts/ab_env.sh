#!/bin/bash
# Same-box A/B of environment knobs: VARIANTS="name:ENV=V,ENV2=V name2:..." interleaved ROUNDS times.
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
out=gpurun_out/ab_env.txt; : > $out
for r in $(seq ${ROUNDS:-3}); do
  for v in $VARIANTS; do
    name=${v%%:*}; envs=${v#*:}
    env $(echo "$envs" | tr ',' ' ') timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-configs ${BENCH_ARGS:-} > gpurun_out/ab_env_$name.json 2>/dev/null
    python - $name gpurun_out/ab_env_$name.json >> $out <<'PY'
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
