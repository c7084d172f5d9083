#!/bin/bash
# Iteration loop on one GPU box: build, GPU tests, instrumented GRU kernel
# (diag 5 cycle counters), cache-off kernel timing, default bench line.
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [[ "${SKIP_TESTS:-0}" != 1 ]]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
RNNLM_TC_DIAG=5 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --sessions 8 --no-cache ${BENCH_ARGS:-} 2>&1 | grep prof | tail -1
DIAGS="0" DIAG_ARGS="--sessions 8 --no-cache ${BENCH_ARGS:-}" bash scripts/diag_tc.sh
timeout 600 python bench.py --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('bench', d['value']/1e6, 'Mq/s', d['roofline']['achieved'], d['roofline']['frac'], d['kernel_ms_per_step'])"
