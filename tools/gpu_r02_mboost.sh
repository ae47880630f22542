#!/bin/bash
# A/B: generator cluster boosts through the exact cluster mass (variants/mb) vs make_frame_fast + boost_fma
cd "$(dirname "$0")/.."
HK_LIB_PATH=variants/mb/libhepkit_cuda.so timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_parity_pins_gpu.py tests/test_reference_api.py tests/test_jit_gpu.py 2>&1 | tail -3
for rep in 1 2 3; do for lib in default mb; do for rng in reference philox; do
  if [ "$lib" = default ]; then timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /";
  else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng --chain | sed "s/^{/{\"rng\": \"$rng\", /"; fi
done; done; done 2>&1 | tee gpurun_out/gen_mboost_ab.jsonl
