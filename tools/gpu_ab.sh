#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_1711_05683_b200/libhepkit_cuda.so tools/libhk_mb3.so tools/libhk_mb4.so; do
  HK_LIB_PATH=$PWD/$lib timeout 300 python tools/bench_gen.py --check >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/ab.jsonl; tail -3 gpurun_out/pytest_gpu.log
