#!/bin/bash
# select-free kFcnFast: FCN parity tests, kernel timing at wave sizes and 1e7, call paths
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py tests/test_gpu_parity.py tests/test_parity_pins_gpu.py tests/test_determinism_gpu.py tests/test_splot_gpu.py tests/test_dist_gloo.py 2>&1 | tail -3
for n in 4096 2424832 9699328 10000000 20000000 50000000; do timeout 120 python tools/fcn_fast_time.py $n; done 2>&1 | tee gpurun_out/fcn_fastb_kernel.jsonl
timeout 300 python tools/fcn_many.py | tee gpurun_out/fcn_fastb_many.json
