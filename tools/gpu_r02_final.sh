#!/bin/bash
# Round-end style check: smoke, the GPU suite twice (flakiness), default bench line, reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/pytest_gpu_$i.log 2>&1; echo "pytest $i rc=$?"; tail -2 gpurun_out/pytest_gpu_$i.log; done
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_final.json").read().strip().splitlines()[-1])
print(d["value"], d["roofline"]["frac"], d["clocks"], d["fcn"]["value"], d["fcn"]["roofline"])
PY
