#!/bin/bash
# A/B of the persistent TMA FCN against k_nll_fused<kFcnFast> (variants/notma)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py -k "tma or many or session" 2>&1 | tail -5
for n in 1e7 5e6 2e7 5e7; do
  for lib in default variants/notma/libhepkit_cuda.so; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=$lib timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done 2>&1 | tee gpurun_out/fcn_tma_ab.jsonl
