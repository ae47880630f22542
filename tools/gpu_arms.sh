#!/bin/bash
# Both bench arms as the driver runs them (N=1), plus the torchrun launch path.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?" >> gpurun_out/ref.err
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "ours rc=$?" >> gpurun_out/bench_default.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 10 --warmup 3 --no-fcn --no-cpu > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo "torchrun rc=$?" >> gpurun_out/bench_torchrun.err
tail -1 gpurun_out/ref.err gpurun_out/bench_default.err gpurun_out/bench_torchrun.err
