#!/bin/bash
# always-reverse FCN scan vs alternating, across sizes; batched pass orders
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for n in 2424832 5e6 7e6 1e7 1.5e7 2e7 5e7; do
  for lib in default rev; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done
done 2>&1 | tee gpurun_out/fcn_rev_ab.jsonl
for lib in default rev revmany; do
  if [ "$lib" = default ]; then timeout 300 python tools/fcn_many.py; else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 300 python tools/fcn_many.py; fi
done 2>&1 | tee gpurun_out/fcn_rev_many.jsonl
