#!/bin/bash
# Phase lag (RNNLM_TC_LAG, in 128-row M-tiles) of the fused GRU kernel, interleaved runs.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$1 %.1f Mq/s %.1f us gru %.1f' % (d['value']/1e6, d['ms_per_step']*1e3, k['ms_gru_phase1']*1e3))"; }
for rep in 1 2 3; do for lag in ${LAGS:-32 48 64 96 128}; do RNNLM_TC_LAG=$lag b "lag$lag"; done; done
