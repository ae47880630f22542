#!/bin/bash
# A/B: persistent generator/chain grids (HK_GEN_WAVES / HK_CHAIN_WAVES) vs one CTA per unit
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
HK_LIB_PATH=variants/w1/libhepkit_cuda.so timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_determinism_gpu.py 2>&1 | tail -1
for rep in 1 2 3; do
for lib in default variants/w1/libhepkit_cuda.so variants/w2/libhepkit_cuda.so variants/w8/libhepkit_cuda.so; do
  for rng in reference philox; do
    if [ "$lib" = default ]; then timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /";
    else HK_LIB_PATH=$lib timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /"; fi
  done
done
done 2>&1 | tee gpurun_out/gen_waves_ab.jsonl
