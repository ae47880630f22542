#!/bin/bash
# A/B: fused chain CTA shape (HK_CHAIN_T / ILP / MINB variants)
cd "$(dirname "$0")/.."
for rep in 1 2 3; do for lib in default t128 t32 ilp1m3; do
  if [ "$lib" = default ]; then timeout 120 python tools/bench_gen.py --n 1e7 --reps 5 --chain | sed "s/^{/{\"v\": \"$lib\", /";
  else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/bench_gen.py --n 1e7 --reps 5 --chain | sed "s/^{/{\"v\": \"$lib\", /"; fi
done; done 2>&1 | tee gpurun_out/chain_t_ab.jsonl
