#!/bin/bash
# probes: L2 evict_last loads / scan direction for the FCN column (time + steady-state L2 hits)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for lib in default nf rev ld1 ld2 ld1nf; do
  if [ "$lib" = default ]; then timeout 120 python tools/fcn_fast_time.py 1e7; else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/fcn_fast_time.py 1e7; fi
done
done 2>&1 | tee gpurun_out/fcn_ld_ab.jsonl
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for lib in rev ld1 ld1nf; do
  echo "lib=$lib"
  HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 600 ncu --cache-control none --clock-control none --metrics $M -k regex:k_nll_fused -s 60 -c 4 --csv \
    python tools/fcn_fast_time.py 1e7 2>/dev/null | grep -E "k_nll_fused" | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done | tee gpurun_out/fcn_ld_l2.txt
