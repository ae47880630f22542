#!/bin/bash
# A/B: generator CTAs per SM after the cluster-mass boosts (HK_GEN_T_MINB 4 = product, 5 = variant)
cd "$(dirname "$0")/.."
for rep in 1 2 3; do for v in default minb5; do for rng in reference philox; do
  if [ $v = default ]; then L=""; else L="variants/$v/libhepkit_cuda.so"; fi
  HK_LIB_PATH=$L timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng | sed "s/^{/{\"v\": \"$v\", /"
done; done; done | tee gpurun_out/gen_minb_ab.jsonl
