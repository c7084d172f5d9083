#!/bin/bash
# ncu --set full of the fused GRU kernel on the bench step (MATH: bf16x3 default)
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
M=${MATH:-bf16x3}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_gru_tc' -s ${SKIP:-30} -c 1 \
  -o gpurun_out/prof_gru_${M} -f python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-configs --also none --math $M \
  > gpurun_out/ncu_gru_${M}.log 2>&1
ls -la gpurun_out/prof_gru_${M}.ncu-rep
