#!/bin/bash
# Turn a tools/gpu_evidence.sh + tools/gpu_fp64.sh run (gpurun_out/) into the
# committed evidence under profiles/: bench lines, ncu summary of the
# generator, its DRAM traffic, SASS profile, launch list and FP64 roofline.
set -e
cd "$(dirname "$0")/.."
TAG=${1:-r01}
O=gpurun_out
cp $O/bench_final.json profiles/${TAG}_bench_final.json
[ -s $O/bench_ref.json ] && cp $O/bench_ref.json profiles/${TAG}_bench_reference_arm.json
python tools/ncu_summary.py $O/gen_full.ncu-rep | head -5 > /tmp/ncu_sum.txt
ncu -i $O/gen_full.ncu-rep --page details 2>/dev/null | grep -E "Memory Throughput|DRAM Throughput|Duration|Compute \(SM\) Throughput|Executed Ipc|Issue Slots Busy|SM Busy|L2 Hit Rate|Registers Per|Theoretical Occ|Achieved Occ" > /tmp/ncu_det.txt
{ echo "# ncu --set full --clock-control none --import-source on, k_generate<3,REF,vec2>, 1e8 events (tools/gpu_evidence.sh)"; cat /tmp/ncu_sum.txt /tmp/ncu_det.txt; } > profiles/${TAG}_ncu_generate_full.txt
TAG=$TAG python - <<'PY'
import json, os, re
t = open('/tmp/ncu_sum.txt').read()
rd = float(re.search(r'dram_rd=([\d.]+)Kbyte', t).group(1)) * 1e3
wr = float(re.search(r'dram_wr=([\d.]+)Gbyte', t).group(1)) * 1e9
name = t.split(" | ")[0].strip()
d = {"kernel": name, "events_per_launch": 100000000, "dram_bytes_read": rd,
     "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": 1.04e10,
     "traffic_over_algorithmic": (rd + wr) / 1.04e10,
     "source": "ncu --set full --clock-control none, tools/gpu_evidence.sh (profiles/" + os.environ["TAG"] + "_ncu_generate_full.txt)"}
json.dump(d, open('profiles/generate_traffic.json', 'w'), indent=1)
PY
ncu -i $O/gen_full.ncu-rep --page source --csv --kernel-name regex:k_generate --launch-count 1 --print-source sass > /tmp/s.csv 2>/dev/null
{ echo "SASS-level profile of k_generate<3,REF,vec2> (ncu --set full --import-source, 1e8 events per launch, one launch: per-event counts are per 3-body event)"; python tools/ncu_sass_profile.py /tmp/s.csv 1e8; } > profiles/${TAG}_generate_sass_profile.txt
cp $O/launches.csv profiles/${TAG}_launches.csv
python tools/summarize_launches.py profiles/${TAG}_launches.csv > profiles/${TAG}_launches_summary.txt
python tools/fp64_roofline.py $O/dp_counts.csv $O/fp64_peak.jsonl $TAG > /dev/null
echo "refreshed profiles/ ($TAG)"
