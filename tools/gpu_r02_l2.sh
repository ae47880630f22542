#!/bin/bash
# Steady-state L2 behaviour of the FCN kernel (no cache flush between launches)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
for n in 1e7 5e6 2e6; do
  timeout 600 ncu --cache-control none --clock-control none --metrics $M -k regex:k_nll_fused -s 60 -c 3 --csv \
    python tools/fcn_fast_time.py $n 2>/dev/null | grep -E "k_nll_fused" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tr -d '"'
done | tee gpurun_out/fcn_l2.txt
