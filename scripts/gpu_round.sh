#!/bin/bash
# One GPU session: build, smoke, GPU tests, bench (clean), ncu launch list, ncu full capture
# of the top kernels.  Everything lands in gpurun_out/ (merged back by gpurun).
# usage: bash scripts/gpu_round.sh [tests|bench|ncu|all] [extra bench args...]
set -u
what=${1:-all}; shift || true
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [[ $what == tests || $what == all ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if [[ $what == bench || $what == all ]]; then
  timeout 900 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [[ $what == ncu || $what == all ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_launch_bench.json 2> gpurun_out/ncu_launch.err
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_resolve_parents|k_qcache|k_hcache|k_scan|k_commit|k_gather_a1|k_final|k_gru_tc|k_score|k_dup_scores' -s 430 -c 10 \
    -o gpurun_out/prof_full -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
