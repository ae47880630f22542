#!/bin/bash
# FCN kernel time against whole waves of 592 tiles (148 SMs x 4 CTAs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for n in 4096 606208 1212416 2424832 4849664 7274496 9699328 10000000 12124160 14548992; do
  timeout 120 python tools/fcn_fast_time.py $n
done 2>&1 | tee gpurun_out/fcn_waves.jsonl
