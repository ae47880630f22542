#!/bin/bash
# Round-end evidence on one B200: default bench line, the ncu launch list of
# the headline command, and one ncu --set full capture of the generator.
# Each ncu pass runs only after the same command exited 0 without ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench rc=$?"
B="python bench.py --steps 3 --warmup 3 --no-fcn --no-cpu --no-configs --no-peaks"
timeout 600 $B > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
P="python tools/bench_gen.py --n 1e8 --reps 2"
timeout 300 $P > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_generate' -s 1 -c 1 \
      -o gpurun_out/gen_full -f $P > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
