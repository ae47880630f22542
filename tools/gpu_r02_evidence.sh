#!/bin/bash
# Round-2 evidence bundle on one B200 (each ncu pass only after its command
# exited 0 without ncu): FP64 peak + DP counts, default bench + reference
# arm, launch list, ncu --set full of the generator, C3 chain, Philox
# generator and FCN.  The .ncu-rep files are summarised on the box (text
# under gpurun_out/prof/) and deleted, so the pull stays under 64 MiB.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/prof
bash tools/gpu_fp64.sh
# the bench's FP64 rooflines read the DP counts of the kernels being measured
python tools/fp64_roofline.py gpurun_out/dp_counts.csv gpurun_out/fp64_peak.jsonl r02 > /dev/null
bash tools/gpu_evidence.sh
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
bash tools/gpu_r02_ncu.sh > /dev/null
bash tools/refresh_profiles.sh r02 && cp profiles/r02_* profiles/generate_traffic.json gpurun_out/prof/
for spec in chain_full:2.5e7 gen_philox_full:5e7 fcn_full:1e7 gen_full:1e8; do
  r=${spec%%:*}; ev=${spec##*:}
  [ -f gpurun_out/$r.ncu-rep ] || continue
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/prof/$r.summary.txt
  ncu -i gpurun_out/$r.ncu-rep --page details > gpurun_out/prof/$r.details.txt 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/prof/$r.raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > /tmp/$r.src.csv 2>/dev/null && \
    python tools/ncu_sass_profile.py /tmp/$r.src.csv $ev > gpurun_out/prof/$r.sass_profile.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
