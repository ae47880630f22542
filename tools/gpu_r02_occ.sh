#!/bin/bash
# A/B: kFcnFast load batch x CTAs/SM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for n in 2424832 10000000; do
  for lib in default variants/b16m5 variants/b8m5 variants/b8m6 variants/b4m6 variants/b8m8; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=$lib/libhepkit_cuda.so timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done
done 2>&1 | tee gpurun_out/fcn_occ_ab.jsonl
