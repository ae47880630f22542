"""Compose a committed ncu summary (profiles/rNN_ncu_*.txt) from the text that
tools/gpu_r02_evidence.sh leaves under gpurun_out/prof/ for one capture:
<stem>.summary.txt (tools/ncu_summary.py), <stem>.details.txt (--page details),
<stem>.sass_profile.txt (tools/ncu_sass_profile.py) and <stem>.raw.csv
(--page raw --csv, for the PC-sampling stall reasons).

usage: python tools/compose_ncu.py gpurun_out/prof/gen_philox_full "title" profiles/r02_ncu_generate_philox.txt
"""
import csv
import re
import sys

KEEP = re.compile(r"Memory Throughput|DRAM Throughput|Duration|Compute \(SM\) Throughput|Executed Ipc Active|"
                  r"Issue Slots Busy|L2 Hit Rate|Registers Per|Achieved Occ")


def main(stem, title, out):
    lines = [f"# {title}", open(stem + ".summary.txt").read().strip(), ""]
    seen = set()
    for ln in open(stem + ".details.txt"):
        key = tuple(re.split(r"\s{2,}", ln.strip())[:2])
        if KEEP.search(ln) and key not in seen:
            seen.add(key)
            lines.append(ln.rstrip())
    lines += ["", open(stem + ".sass_profile.txt").read().rstrip(), ""]
    rows = list(csv.reader(open(stem + ".raw.csv")))
    head, vals = rows[0], rows[2]
    stalls = {}
    for i, name in enumerate(head):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"):
            try:
                stalls[name] = float(vals[i].replace(",", ""))
            except ValueError:
                pass
    total = sum(stalls.values()) or 1.0
    lines.append("stall reasons (share of samples):")
    for name, v in sorted(stalls.items(), key=lambda kv: -kv[1]):
        if v / total >= 0.005:
            lines.append(f"  {100 * v / total:5.1f}% {name}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
