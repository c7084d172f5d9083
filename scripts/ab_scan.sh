#!/bin/bash
# Look-back scan tile size (-DRNNLM_SCAN_ITEMS: queries per thread, 256 threads per tile).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
b() { timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$1 %.1f Mq/s %.1f us cache %.1f' % (d['value']/1e6, d['ms_per_step']*1e3, k['ms_cache']*1e3))"; }
for rep in 1 2; do for it in ${ITEMS:-1 2 4 8}; do
  RNNLM_NVCC_FLAGS=-DRNNLM_SCAN_ITEMS=$it python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1
  b "items$it"
done; done
for it in 4 8; do
  RNNLM_NVCC_FLAGS=-DRNNLM_SCAN_ITEMS=$it python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1
  timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fullsize or multi_config or edge or ragged or unsorted" 2>&1 | tail -1
done
python -c "from paper_1801_09866_b200 import build; build.build(force=True)" > /dev/null 2>&1
