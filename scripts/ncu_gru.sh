#!/bin/bash
# ncu --set full on the GRU GEMM kernels only (one launch each, mid-run)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gru1_tc|k_gru2_tc|k_gather_a1' -s 60 -c 3 \
  -o gpurun_out/prof_gru -f python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_gru.log 2>&1
tail -3 gpurun_out/ncu_gru.log
