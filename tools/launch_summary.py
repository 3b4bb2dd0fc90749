"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:90]
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
    total += v
unit = hdr[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
print(f"{'kernel':92s} {'launches':>8s} {'total':>12s} {'share':>7s}")
for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name:92s} {c:8d} {t:12.0f} {100 * t / total:6.1f}%")
print(f"total {sum(c for c, _ in agg.values())} launches, {total:.0f} (ns) summed device time")
