#!/bin/bash
# Steady-state L2 hit rate of the FCN kernel with the alternating scan direction
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for n in 1e7 7e6; do
  echo "n=$n"
  timeout 600 ncu --cache-control none --clock-control none --metrics $M -k regex:k_nll_fused -s 60 -c 4 --csv \
    python tools/fcn_fast_time.py $n 2>/dev/null | grep -E "k_nll_fused" | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done | tee gpurun_out/fcn_l2_flip.txt
