#!/bin/bash
# A/B of the RNG software pipeline in k_generate (HK_GEN_PIPE variants) on both
# streams, the Philox/generator parity tests, and the nll() host-overhead probe.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_parity_pins_gpu.py tests/test_determinism_gpu.py 2>&1 | tail -3
for rep in 1 2; do
for lib in default variants/pipe0/libhepkit_cuda.so variants/pipe1/libhepkit_cuda.so variants/pipe3/libhepkit_cuda.so; do
  for rng in reference philox; do
    if [ "$lib" = default ]; then timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng | sed "s/^{/{\"rng\": \"$rng\", /";
    else HK_LIB_PATH=$lib timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 --rng $rng | sed "s/^{/{\"rng\": \"$rng\", /"; fi
  done
done
done 2>&1 | tee gpurun_out/gen_pipe_ab.jsonl
timeout 300 python tools/fcn_py_overhead.py > gpurun_out/fcn_py_overhead.json 2>&1; cat gpurun_out/fcn_py_overhead.json
