#!/bin/bash
# GRU kernel timing at a fixed all-miss size (8 sessions x 2048 rows, cache off):
# full kernel, diag modes (see k_gru_tc.cu TcArgs::diag), cycle counters (diag 5);
# one-CTA (PAIRS=0) and CTA-pair (PAIRS=1) kernels.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in ${PAIRS:-0 1}; do
for d in ${DIAGS:-0 6 3}; do
  RNNLM_TC_PAIR=$p RNNLM_TC_DIAG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --sessions 8 --no-cache --timing-level 2 ${BENCH_ARGS:-} > /tmp/o.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']; print('pair $p diag $d gru %.1f us' % (k['ms_gru_phase1']*1e3))"
done
RNNLM_TC_PAIR=$p RNNLM_TC_DIAG=5 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --sessions 8 --no-cache ${BENCH_ARGS:-} 2>&1 | grep prof | tail -1
done
