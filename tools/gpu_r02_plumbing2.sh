#!/bin/bash
# N=2 code path of the full bench (secondary configs, FCN, CPU baseline off) with gloo ranks sharing one GPU
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
HK_BENCH_BACKEND=gloo HK_BENCH_DEVICE=0 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu \
  > gpurun_out/plumb2_n2.json 2> gpurun_out/plumb2_n2.err; echo "N=2 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/plumb2_n2.json').read().strip().splitlines()[-1])
print(d['n_gpus'], d['value'], sorted((d.get('other_configs') or {}).keys()), (d.get('fcn') or {}).get('value'))"
tail -3 gpurun_out/plumb2_n2.err
