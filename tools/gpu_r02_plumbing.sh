#!/bin/bash
# N>1 code path of bench.py with gloo ranks sharing one GPU (plumbing check only, never a bench number)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for N in 2 4; do
  HK_BENCH_BACKEND=gloo HK_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --steps 3 --warmup 3 --no-cpu --no-configs \
    > gpurun_out/plumb_n$N.json 2> gpurun_out/plumb_n$N.err; echo "N=$N rc=$?"
  tail -c 600 gpurun_out/plumb_n$N.json; echo; tail -3 gpurun_out/plumb_n$N.err
done
