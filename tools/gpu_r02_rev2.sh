#!/bin/bash
# FCN scan-direction policy: threshold sweep around 0.75 x L2, then the product default
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_fcn_generic_gpu.py tests/test_determinism_gpu.py 2>&1 | tail -1
for n in 1e7 1.1e7 1.2e7 1.3e7 1.5e7; do
  for thr in 0 200000000; do HK_FCN_REV_MAX_BYTES=$thr timeout 120 python tools/fcn_fast_time.py $n | sed "s/^{/{\"rev_max\": $thr, /"; done
done 2>&1 | tee gpurun_out/fcn_rev_thr.jsonl
for n in 5e6 1e7 1.5e7 2e7 5e7; do timeout 120 python tools/fcn_fast_time.py $n; done 2>&1 | tee gpurun_out/fcn_rev_default.jsonl
timeout 300 python tools/fcn_many.py | tee gpurun_out/fcn_many_rev.json
