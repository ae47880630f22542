#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "unweight or where or select or compact" 2>&1 | tail -1
timeout 300 python tools/unweight_time.py | tee gpurun_out/unweight.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_unweight|k_scan|k_compact" -c 6 --csv python tools/unweight_time.py 1e8 2>/dev/null | grep -E "k_unweight|k_scan|k_compact" | awk -F'","' '{print $5, $NF}' | tr -d '"' | tail -6
