#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; rm -f gpurun_out/ab.jsonl
for lib in paper_1711_05683_b200/libhepkit_cuda.so tools/libhk_*.so; do
  HK_LIB_PATH=$PWD/$lib timeout 300 python tools/bench_gen.py --check >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
done
timeout 300 python tools/fcn_overhead.py >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
cat gpurun_out/ab.jsonl
