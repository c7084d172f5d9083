#!/bin/bash
# ncu --set full on the fused GRU kernel + gather at a timed (mid-utterance) frame
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gru_tc|k_gather_a1' -s 84 -c 2 \
  -o gpurun_out/prof_gru -f python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_gru.log 2>&1
tail -3 gpurun_out/ncu_gru.log
