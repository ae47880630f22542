#!/bin/bash
# A/B: FCN scan direction alternating per call (L2 reuse across calls) vs fixed (variants/noflip)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py tests/test_gpu_parity.py tests/test_parity_pins_gpu.py tests/test_determinism_gpu.py tests/test_splot_gpu.py 2>&1 | tail -1
for rep in 1 2; do
for n in 1e7 2e7 5e7; do
  for lib in default variants/noflip/libhepkit_cuda.so; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=$lib timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done
done 2>&1 | tee gpurun_out/fcn_flip_ab.jsonl
for lib in default variants/noflip/libhepkit_cuda.so; do
  if [ "$lib" = default ]; then timeout 300 python tools/fcn_many.py; else HK_LIB_PATH=$lib timeout 300 python tools/fcn_many.py; fi
done 2>&1 | tee gpurun_out/fcn_flip_many.jsonl
