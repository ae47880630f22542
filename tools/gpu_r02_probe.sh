#!/bin/bash
# Round-2 measurement probe: FCN latency paths, HBM write peaks, Philox and C3 generator rates.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/store_pattern.cu -o /tmp/store_pattern && /tmp/store_pattern > gpurun_out/store_pattern.jsonl 2>&1
timeout 300 python tools/peak_write.py > gpurun_out/peak_write.json 2>&1
timeout 300 python tools/bench_gen.py --n 1e8 --reps 10 --chain > gpurun_out/gen_ref.json 2>&1
timeout 300 python tools/bench_gen.py --n 1e8 --reps 10 --chain --rng philox > gpurun_out/gen_philox.json 2>&1
timeout 600 python tools/fcn_many.py > gpurun_out/fcn_many.json 2>&1
timeout 300 python tools/fcn_session_probe.py > gpurun_out/fcn_session.json 2>&1
tail -n 3 gpurun_out/*.json gpurun_out/*.jsonl
