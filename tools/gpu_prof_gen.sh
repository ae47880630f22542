#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P="python tools/bench_gen.py --n 1e8 --reps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_generate|k_nll_fused' -s 1 -c 3 \
      -o gpurun_out/gen_full -f $P > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
