#!/bin/bash
# A/B: constant-bank math coefficients in the generator (variants/cbank)
cd "$(dirname "$0")/.."
for rep in 1 2 3; do for lib in default cbank; do for rng in reference philox; do
  if [ "$lib" = default ]; then timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /";
  else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /"; fi
done; done; done 2>&1 | tee gpurun_out/gen_cbank_ab.jsonl
