#!/bin/bash
# iterate: gpu tests, kernel microbench, bench line, ncu full capture of hot kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_gen.py --check > gpurun_out/gen.json 2>&1
timeout 900 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ -n "$PROF" ]; then
  P="python tools/prof_kernels.py"
  $P > gpurun_out/prof_plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:"$PROF" -s ${PROF_SKIP:-1} -c ${PROF_COUNT:-4} \
        -o gpurun_out/${PROF_OUT:-kernels_full} -f $P > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/gen.json; tail -1 gpurun_out/bench.err
