"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name, launches / total / mean time and share of GPU time."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit_i = hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[unit_i]]
    tot[r[ki]] += v * scale
    cnt[r[ki]] += 1
allt = sum(tot.values())
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{cnt[k]:5d} launches {tot[k] / 1e3:10.3f} ms total {tot[k] / cnt[k]:10.1f} us/launch "
          f"{100 * tot[k] / allt:6.2f}% of GPU time  {k}")
