#!/bin/bash
# A/B: the persistent TMA FCN at every size vs k_nll_fused at 1e7, warm (back to back) and after an L2 flush
cd "$(dirname "$0")/.."
for rep in 1 2; do for v in default tma_all; do
  if [ $v = default ]; then L=""; else L="variants/$v/libhepkit_cuda.so"; fi
  HK_LIB_PATH=$L timeout 300 python bench.py --no-cpu --no-configs 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); f=d['fcn']
print(json.dumps({'v': '$v', 'fcn': f['value'], 'kernel_us': f['kernel_us'], 'kernel_us_l2_flushed': f['kernel_us_l2_flushed'], 'session': f['session_evals_per_s'], 'batched51': f['batched51_evals_per_s']}))"
done; done | tee gpurun_out/fcn_tma_cold_ab.jsonl
