#!/bin/bash
# Register cap of the fused GRU kernels (-DGRU_MAXREG), interleaved bench runs.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
b() { timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$1 %.1f Mq/s %.1f us gru %.1f score %.1f' % (d['value']/1e6, d['ms_per_step']*1e3, k['ms_gru_phase1']*1e3, k['ms_score']*1e3))"; }
for rep in 1 2 3; do for r in ${REGS:-144 152 168}; do
  RNNLM_NVCC_FLAGS=-DGRU_MAXREG=$r python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1
  b "maxreg$r"
done; done
python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1
