#!/bin/bash
# ncu launch list of the bench's timed step command (no write-peak fills)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-fcn --no-cpu --no-configs --no-peaks"
timeout 600 $B > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
