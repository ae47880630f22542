#!/bin/bash
# A/B: FCN ticket as one acq_rel RMW (variants/acqrel) vs __threadfence + atomicAdd
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
HK_LIB_PATH=variants/acqrel/libhepkit_cuda.so timeout 900 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py tests/test_determinism_gpu.py tests/test_gpu_parity.py -k "nll or fcn or determin or shard" 2>&1 | tail -1
for rep in 1 2; do
for n in 4096 2424832 10000000; do
  for lib in default variants/acqrel/libhepkit_cuda.so; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=$lib timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done
done 2>&1 | tee gpurun_out/fcn_acqrel_ab.jsonl
