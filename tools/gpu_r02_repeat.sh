#!/bin/bash
# the default bench line three times on one box (run-to-run spread)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu --no-configs 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(json.dumps({'run': $i, 'value': d['value'], 'frac': d['roofline']['frac'], 'e2e': d['e2e']['value'], 'fcn': d['fcn']['value'], 'fcn_kernel_us': d['fcn']['kernel_us'], 'session': d['fcn']['session_evals_per_s'], 'batched51': d['fcn']['batched51_evals_per_s']}))"
done | tee gpurun_out/bench_repeat.jsonl
