#!/bin/bash
# A/B: k_compact column load grouping (HK_COMPACT_GROUP: default 8, variants 0/4/16)
cd "$(dirname "$0")/.."
timeout 600 python -m pytest -q -x -m gpu tests -k "unweight or compact or where_mask or select" 2>&1 | tail -1
for rep in 1 2; do for v in default cg0 cg4 cg16; do
  if [ $v = default ]; then timeout 120 python tools/unweight_time.py 1e8 | sed "s/^{/{\"v\": \"$v\", /";
  else HK_LIB_PATH=variants/$v/libhepkit_cuda.so timeout 120 python tools/unweight_time.py 1e8 | sed "s/^{/{\"v\": \"$v\", /"; fi
done; done | tee gpurun_out/compact_ab.jsonl
