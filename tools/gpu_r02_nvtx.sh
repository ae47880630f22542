#!/bin/bash
# NVTX ranges: smoke + a GPU test subset, then ncu selecting the FCN kernel by its C-ABI range
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_fcn_generic_gpu.py tests/test_csv_gpu.py 2>&1 | tail -1
timeout 600 ncu --nvtx --nvtx-include "hk_nll_eval/" --metrics gpu__time_duration.sum --clock-control none -c 3 \
   python tools/fcn_fast_time.py 1e7 2>&1 | grep -E "k_nll|hk_nll_eval|NVTX|==PROF==" | head -12 | tee gpurun_out/nvtx_ncu.txt
