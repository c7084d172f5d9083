#!/bin/bash
# Memory kernels of the bench step under ncu on the uniform-word stream (no Zipf
# reuse: DRAM bytes ~ algorithmic bytes) and on the Zipf stream, bf16 step.
# Summarised by scripts/mem_summary.py into profiles/.
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-configs --also none"
MM="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_sector_hit_rate.pct"
K='k_gather_a1|k_score|k_qcache|k_hcache|k_scan|k_commit|k_final|k_dup_scores'
timeout 900 ncu --metrics $MM --clock-control none -k regex:"$K" -s 3000 -c 40 --csv \
  --log-file gpurun_out/ncu_uniform_r2.csv $B --math bf16 --uniform-words > gpurun_out/ncu_uniform_bench.json 2> gpurun_out/ncu_uniform.err
timeout 900 ncu --metrics $MM --clock-control none -k regex:"$K" -s 3000 -c 40 --csv \
  --log-file gpurun_out/ncu_zipf_r2.csv $B --math bf16 > /dev/null 2> gpurun_out/ncu_zipf.err
ls -la gpurun_out
