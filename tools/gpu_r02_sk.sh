#!/bin/bash
# A/B: compile-time decaying daughter in the fused C3 chain (variants/sk)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
HK_LIB_PATH=variants/sk/libhepkit_cuda.so timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_parity_pins_gpu.py -k "chain" 2>&1 | tail -1
for rep in 1 2 3; do
  for lib in default sk; do
    for rng in reference philox; do
      if [ "$lib" = default ]; then timeout 120 python tools/bench_gen.py --n 1e8 --reps 10 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /";
      else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/bench_gen.py --n 1e8 --reps 10 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /"; fi
    done
  done
done 2>&1 | tee gpurun_out/chain_sk_ab.jsonl
