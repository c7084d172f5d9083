#!/bin/bash
# One-CTA kernel ring depth (-DRNNLM_TC_ST) on its workloads (TF32, LBR, RNN)
# and the pair kernel's phase lag (RNNLM_TC_LAG) on the default workload.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
b() { timeout 300 python bench.py --no-e2e --no-cpu-baseline $2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$1 %.1f Mq/s %.1f us gru %.1f' % (d['value']/1e6, d['ms_per_step']*1e3, k['ms_gru_phase1']*1e3))"; }
python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1
for lag in 32 64 128 256; do RNNLM_TC_LAG=$lag b "lag$lag" ""; done
for rep in 1 2; do
  for st in 3 4; do
    RNNLM_NVCC_FLAGS=-DRNNLM_TC_ST=$st python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1
    b "st$st tf32" "--math tf32"; b "st$st lbr" "--cell lbr"; b "st$st rnn" "--cell rnn"
  done
done
python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1
