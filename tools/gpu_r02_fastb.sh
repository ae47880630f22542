#!/bin/bash
# timing probe: select-free kFcnFast (density normalised by the exponential term) vs current
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for n in 4096 2424832 9699328 10000000; do
  for lib in default variants/fastb/libhepkit_cuda.so; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=$lib timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done
done 2>&1 | tee gpurun_out/fcn_fastb_ab.jsonl
