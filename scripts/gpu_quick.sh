#!/bin/bash
# Quick GPU iteration: build, a pytest selection (-k $K), then bench lines (BENCH_ARGS).
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
if [[ -n "${K:-}" ]]; then
  timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$K" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
  tail -4 gpurun_out/pytest_quick.log
fi
if [[ -n "${BENCH_ARGS:-}" ]]; then
  timeout 900 python bench.py $BENCH_ARGS > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?" >> gpurun_out/bench_quick.err
  python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1])
def show(tag,x):
    r=x['roofline']; print(tag, round(x['value']/1e6,1),'Mq/s', 'ms/step',round(x['ms_per_step'],4), 'kernel ms',round(r['kernel_ms_per_step'],4), 'ach',round(r['achieved'],1),'peak',round(r['peak'],1),'frac',round(r['frac'],3), 'ms',{k:round(v,4) for k,v in x['kernel_ms_per_step'].items()})
show(d['config']['math'], d)
for k in ('bf16','tf32x3','bf16x3','tf32','fp32'):
    if k in d and isinstance(d[k],dict): show(k,d[k])
PY
fi
