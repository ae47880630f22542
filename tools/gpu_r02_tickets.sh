#!/bin/bash
# A/B: hierarchical CTA tickets (variants/t4, t8) vs one flat ticket
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
HK_LIB_PATH=variants/t8/libhepkit_cuda.so timeout 900 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py tests/test_determinism_gpu.py tests/test_gpu_parity.py -k "nll or fcn or determin or shard" 2>&1 | tail -1
timeout 900 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py -k "session or many or regimes" 2>&1 | tail -1
for rep in 1 2 3; do
for n in 2424832 10000000; do
  for lib in default t4 t8; do
    if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py $n; else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/fcn_fast_time.py $n; fi
  done
done
done 2>&1 | tee gpurun_out/fcn_tickets_ab.jsonl
