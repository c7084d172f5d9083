#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
for r in 1 2; do for v in a b; do
  lib=paper_1801_09866_b200/librnnlm.so; [[ $v == a ]] && lib=paper_1801_09866_b200/librnnlm_a.so
  RNNLM_LIBRARY=$PWD/$lib timeout 600 python bench.py --no-e2e --no-cpu-baseline --also none --steps 5 --warmup 3 > gpurun_out/abs_$v.json 2>/dev/null
  python - $v gpurun_out/abs_$v.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
out = []
for name in ("tiny", "moderate"):
    for k, v in d["configs"][name]["results"].items():
        out.append("%s/%s %.1f us (kernel %.1f)" % (name, k, v["us_per_frame"], v["fused_kernel"]["us_per_frame"]))
print(sys.argv[1], " | ".join(out))
PY
done; done
