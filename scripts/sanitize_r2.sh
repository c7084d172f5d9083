#!/bin/bash
# compute-sanitizer over the round-2 additions (BF16X3 on both CTA shapes, the fused
# small-frame kernel, graphs, normaliser with off-grid rows, one-session full-size replay)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
K1="bf16x3_moderate or bf16x3_large or bf16x3_skips or test_tiny_config_fused or fused_edge or fused_graph or off_grid_output or edge_cases_invalid"
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K1" > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
K2="bf16x3_moderate_fp32_tolerance or test_tiny_config_fused or fused_edge"
timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K2" > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
tail -5 gpurun_out/sanitize_memcheck.log gpurun_out/sanitize_racecheck.log
