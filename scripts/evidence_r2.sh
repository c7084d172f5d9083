#!/bin/bash
# Round-2 evidence: compression sweeps (BASELINE configs[3], and the moderate model for
# Table 1's H = 256 shape), the per-query vs per-frame ablation, the offline schedule,
# the log-normaliser, the reference arm.  Outputs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python scripts/sweep.py --what sweep --sessions 8 --frames 400 --math bf16x3 > gpurun_out/sweep_large_r2.jsonl 2> gpurun_out/sweep_large.err
timeout 900 python scripts/sweep.py --what sweep --config moderate --sessions 1 --frames 400 --math bf16x3 > gpurun_out/sweep_moderate_r2.jsonl 2> gpurun_out/sweep_moderate.err
timeout 900 python scripts/sweep.py --what ablation > gpurun_out/ablation_moderate_r2.jsonl 2> gpurun_out/ablation.err
timeout 900 python bench.py --offline --math bf16x3 > gpurun_out/offline_bench_r2.jsonl 2> gpurun_out/offline.err
timeout 900 python bench.py --offline --math bf16x3 --workload moderate >> gpurun_out/offline_bench_r2.jsonl 2>> gpurun_out/offline.err
timeout 900 python bench.py --normalizer > gpurun_out/normalizer_bench_r2.json 2> gpurun_out/normalizer.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/reference_arm_r2.json 2> gpurun_out/reference.err
ls -la gpurun_out
