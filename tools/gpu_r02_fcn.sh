#!/bin/bash
# FCN timing + ncu of the kFcnFast kernels (single-point and 51-point)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/fcn_many.py > gpurun_out/fcn_many.json 2>&1; echo "many rc=$?"
timeout 600 python tools/fcn_session_probe.py > gpurun_out/fcn_session.json 2>&1; echo "probe rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_nll_fused|k_nll_many' -s 10 -c 2 \
    -o gpurun_out/fcn_fast_full -f python tools/fcn_many.py > gpurun_out/ncu_fcn_fast.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/fcn_many.json gpurun_out/fcn_session.json
