#!/bin/bash
# Round-2 evidence bundle on one B200 (each ncu pass only after its command
# exited 0 without ncu): FP64 peak + DP counts, default bench + reference
# arm, launch list, ncu --set full of the generator, C3 chain, Philox
# generator and FCN.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_fp64.sh
python tools/fp64_roofline.py gpurun_out/dp_counts.csv gpurun_out/fp64_peak.jsonl r02 > /dev/null && cp profiles/r02_fp64_roofline.json gpurun_out/
bash tools/gpu_evidence.sh
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
bash tools/gpu_r02_ncu.sh
