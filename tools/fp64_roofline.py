"""FP64 roofline evidence: per-event DP instruction counts of
the hot kernels, from an ncu metrics pass, against the DFMA peak measured by
tools/fp64_peak.cu.  Writes profiles/<round>_fp64_roofline.json.

    # on the box (tools/gpu_fp64.sh): fp64_peak.jsonl + dp_counts.csv into gpurun_out/
    python tools/fp64_roofline.py gpurun_out/dp_counts.csv gpurun_out/fp64_peak.jsonl r01

Every DP instruction (DFMA, DMUL, DADD) occupies one FP64 issue slot, so the
FP64-pipe roofline is DP instructions/s against the measured DFMA
instructions/s; TFLOP/s (DFMA = 2 flops) is reported beside it.
"""

from __future__ import annotations

import csv
import json
import os
import sys

EVENTS = {  # events per launch in tools/prof_kernels.py
    "k_generate<": 100_000_000,
    "hk_jit_integrate": 100_000_000,
    "k_generate_chain<": 50_000_000,
    "k_nll_fused<": 10_000_000,
    "k_nll_many<": 10_000_000 * 52,   # event-points: 52 parameter points per launch
}


def main() -> None:
    counts_csv, peak_jsonl, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    peaks = [json.loads(line) for line in open(peak_jsonl) if line.startswith("{")]
    peak = max(peaks, key=lambda p: p["dfma_per_s"])
    rows = [r for r in csv.reader(open(counts_csv)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches: dict = {}
    for r in rows[1:]:
        launches.setdefault(r[ii], {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    out = {}
    for m in launches.values():
        key = next((k for k in EVENTS if k in m["kernel"]), None)
        if key is None or key in out:
            continue   # first launch of each kernel
        n = EVENTS[key]
        dfma = m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
        dmul = m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
        dadd = m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
        t = m["gpu__time_duration.sum"] * 1e-9
        inst = dfma + dmul + dadd
        out[key.rstrip("<")] = {
            "kernel": m["kernel"], "events_per_launch": n,
            "dp_inst_per_event": inst / n, "dfma_per_event": dfma / n, "dmul_per_event": dmul / n,
            "dadd_per_event": dadd / n, "dp_flops_per_event": (2 * dfma + dmul + dadd) / n,
            "ncu_launch_s": t,
            "dp_inst_frac_of_peak_ncu": inst / t / peak["dfma_per_s"],
            "tflops_ncu": (2 * dfma + dmul + dadd) / t * 1e-12,
            "fp64_pipe_active_pct_ncu": m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
        }
    res = {"peak": {"dp_inst_per_s": peak["dfma_per_s"], "tflops": peak["fp64_tflops"],
                    "sm_clock_mhz_est": peak["sm_clock_mhz_est"],
                    "lanes_per_sm_per_clk": peak["dfma_lanes_per_sm_per_clk"],
                    "source": "measured: tools/fp64_peak.cu (" + peak["how"] + ")"},
           "kernels": out,
           "how": "ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum,"
                  "sm__pipe_fp64_cycles_active,gpu__time_duration --clock-control none over "
                  "tools/prof_kernels.py (cold, serialised launches)"}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "profiles", f"{tag}_fp64_roofline.json")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
