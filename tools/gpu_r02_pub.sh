#!/bin/bash
# FCN publication with plain re-arm (product) vs the previous build: tests + 1e7 / 1-wave timing
cd "$(dirname "$0")/.."
timeout 900 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py tests/test_determinism_gpu.py tests/test_gpu_parity.py -k "nll or fcn or determin or shard or bad" 2>&1 | tail -1
for rep in 1 2 3; do for n in 2424832 10000000; do timeout 120 python tools/fcn_fast_time.py $n; done; done 2>&1 | tee gpurun_out/fcn_pub.jsonl
