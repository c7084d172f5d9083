#!/bin/bash
# Round-2 ncu evidence (B200_PROFILING recipe).  Outputs land in gpurun_out/.
#  1. launch list of the headline bench command (one pass, per-launch duration)
#  2. tensor-pipe / op-count / DRAM counters of the GRU kernels (headline 3xTF32 and bf16)
#  3. one --set full capture of the top kernels of the headline step
#  4. the fused small-frame kernel (moderate config, one stream)
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-configs --also none"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
  $B > gpurun_out/ncu_launch_bench.json 2> gpurun_out/ncu_launch.err
M="gpu__time_duration.sum,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__inst_executed_pipe_tc.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for math in tf32x3 bf16; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:'k_gru_tc' -s 362 -c 3 --csv \
    --log-file gpurun_out/ncu_tensor_${math}.csv $B --math $math > /dev/null 2> gpurun_out/ncu_tensor_${math}.err
done
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:'k_gru_tc|k_gather_a1|k_score|k_qcache|k_hcache|k_scan|k_commit|k_final' -s 3000 -c 10 \
  -o gpurun_out/prof_r2 -f $B > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_small' -s 100 -c 2 \
  -o gpurun_out/prof_small_r2 -f python scripts/latency_probe.py moderate bf16 auto > gpurun_out/ncu_small.log 2>&1
ls -la gpurun_out
# 5. memory kernels on the uniform-word stream (no Zipf reuse: DRAM bytes ~ algorithmic bytes), bf16 step
MM="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_sector_hit_rate.pct"
timeout 900 ncu --metrics $MM --clock-control none -k regex:'k_gather_a1|k_score|k_qcache|k_hcache|k_scan|k_commit|k_final|k_dup_scores' \
  -s 3000 -c 40 --csv --log-file gpurun_out/ncu_uniform_r2.csv $B --math bf16 --uniform-words > gpurun_out/ncu_uniform_bench.json 2> gpurun_out/ncu_uniform.err
timeout 900 ncu --metrics $MM --clock-control none -k regex:'k_gather_a1|k_score|k_qcache|k_hcache|k_scan|k_commit|k_final|k_dup_scores' \
  -s 3000 -c 40 --csv --log-file gpurun_out/ncu_zipf_r2.csv $B --math bf16 > /dev/null 2> gpurun_out/ncu_zipf.err
ls -la gpurun_out
