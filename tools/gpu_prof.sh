#!/bin/bash
# ncu launch list of the bench command + full captures of the hot kernels (one ncu tool per call).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-fcn --no-cpu --no-configs"
$B > gpurun_out/prof_bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
P="python tools/prof_kernels.py"
$P > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_generate|k_integrate|k_nll_fused' -s 2 -c 5 \
      -o gpurun_out/kernels_full -f $P > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -2 gpurun_out/ncu_full.log
