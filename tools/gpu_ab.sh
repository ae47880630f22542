#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; rm -f gpurun_out/ab.jsonl
for lib in paper_1711_05683_b200/libhepkit_cuda.so tools/libhk_*.so; do
  HK_LIB_PATH=$PWD/$lib timeout 300 python tools/bench_gen.py --check >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
done
cat gpurun_out/ab.jsonl
timeout 120 python tools/peak_write.py >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
tail -1 gpurun_out/ab.jsonl
