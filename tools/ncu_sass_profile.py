"""Aggregate an ncu SASS source page: executed instructions and stall samples per opcode.

    ncu -i rep --page source --csv --kernel-name regex:K --launch-count 1 --print-source sass > s.csv
    python tools/ncu_sass_profile.py s.csv [events]
"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
events = float(sys.argv[2]) if len(sys.argv) > 2 else None
hdr = rows[1]
i_src, i_exec, i_samp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
exe, samp = Counter(), Counter()
tot_e = tot_s = 0
top = []
for r in rows[2:]:
    if len(r) <= max(i_samp, i_exec):
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[i_src].strip()).split(" ")[0].split(".")[0]
    try:
        e = float(r[i_exec] or 0)
        s = float(r[i_samp] or 0)
    except ValueError:
        continue
    exe[op] += e
    samp[op] += s
    tot_e += e
    tot_s += s
    top.append((s, r[0], r[i_src].strip()[:70]))
print(f"warp instructions executed: {tot_e:.4g}" + (f"  ({tot_e * 32 / events:.1f} thread-instr/event)" if events else ""))
for op, e in exe.most_common(22):
    extra = f" per-event {e * 32 / events:6.1f}" if events else ""
    print(f"  {op:10s} {e / tot_e * 100:5.1f}% of instr  {samp[op] / max(tot_s, 1) * 100:5.1f}% of stall samples{extra}")
print("top stalled instructions:")
for s, addr, src in sorted(top, reverse=True)[:15]:
    print(f"  {s / tot_s * 100:5.1f}%  {addr}  {src}")
