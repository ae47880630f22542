#!/bin/bash
# A/B of the prefetching persistent kFcnFast FCN (variants/pf<minb>) against k_nll_fused<kFcnFast>
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 2 3 4 5; do HK_LIB_PATH=variants/pf$v/libhepkit_cuda.so timeout 600 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py -k "tma or many" 2>&1 | tail -1; done
for rep in 1 2; do
for n in 1e7 2e6; do
  for lib in default variants/pf2/libhepkit_cuda.so variants/pf3/libhepkit_cuda.so variants/pf4/libhepkit_cuda.so variants/pf5/libhepkit_cuda.so; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=$lib timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done
done 2>&1 | tee gpurun_out/fcn_pf_ab.jsonl
