#!/bin/bash
# CUPTI kernel timeline of a few timed steps (bench.py --trace) + a clean bench line.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --trace gpurun_out/trace.json ${BENCH_ARGS:-} > gpurun_out/trace_bench.json 2>&1
python scripts/timeline.py gpurun_out/trace.json 3
timeout 600 python bench.py --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_trace.json 2> gpurun_out/bench_trace.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_trace.json').read().strip().splitlines()[-1]); print('bench %.1f Mq/s  %.1f us/step  gru %.1f TF frac %.3f' % (d['value']/1e6, d['ms_per_step']*1e3, d['roofline']['achieved'], d['roofline']['frac']))"
