#!/bin/bash
# timing probe: spread-tail FCN schedule (variants/spread) vs plain tiles
cd "$(dirname "$0")/.."
for rep in 1 2 3; do for n in 1e7 5e6; do
  timeout 120 python tools/fcn_fast_time.py $n
  HK_LIB_PATH=variants/spread/libhepkit_cuda.so timeout 120 python tools/fcn_fast_time.py $n
done; done 2>&1 | tee gpurun_out/fcn_spread_ab.jsonl
