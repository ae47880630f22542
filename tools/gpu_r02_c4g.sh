#!/bin/bash
# FCN density-program path (BW + polynomial closures): tests, then timing
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py tests/test_jit_gpu.py tests/test_parity_pins_gpu.py tests/test_splot_gpu.py 2>&1 | tail -1
for rep in 1 2; do timeout 300 python tools/fcn_generic_time.py 2>&1 | tail -1; done | tee gpurun_out/fcn_generic_spt.jsonl
