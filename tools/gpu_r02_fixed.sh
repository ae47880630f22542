#!/bin/bash
# FCN fixed cost probes: empty kernel, no ticket/fold, full kernel
cd "$(dirname "$0")/.."
for n in 4096 606208 2424832 10000000; do
  for lib in default nofin empty; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done 2>&1 | tee gpurun_out/fcn_fixed.jsonl
