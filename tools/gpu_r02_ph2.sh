#!/bin/bash
# A/B: Philox generation with 3 blocks/event (53-bit uniforms, product) vs 2 blocks (51-bit probe)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_parity_pins_gpu.py tests/test_jit_gpu.py 2>&1 | tail -2
for rep in 1 2 3; do
for lib in default variants/ph2/libhepkit_cuda.so; do
  for rng in reference philox; do
    if [ "$lib" = default ]; then timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /";
    else HK_LIB_PATH=$lib timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng | sed "s/^{/{\"rng\": \"$rng\", /"; fi
  done
done
done 2>&1 | tee gpurun_out/gen_ph2_ab.jsonl
