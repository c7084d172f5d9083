cd $GRAFT_REPO_ROOT
for st in 2 3 4; do
  RNNLM_NVCC_FLAGS="-DRNNLM_TC_ST=$st" python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > gpurun_out/st_build$st.log 2>&1
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --timing-level 2 > gpurun_out/st$st.json 2> gpurun_out/st$st.err
done
