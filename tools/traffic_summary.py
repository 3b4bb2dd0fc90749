"""Summarise tools/step_traffic.sh's ncu launch list: per kernel launches,
DRAM bytes (read + write), device time and GB/s; the step total; and a JSON
record (stdout's last line) for profiles/:
  python tools/traffic_summary.py traffic_C2.csv traffic_graph_C2.log C2
"""
import csv
import json
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
idi = hdr.index("ID")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0}
launch = defaultdict(dict)
names = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    launch[r[idi]][r[mi]] = v
    names[r[idi]] = r[ki].split("(")[0]
agg = defaultdict(lambda: [0, 0.0, 0.0])
tb = tt = 0.0
for i, m in launch.items():
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    t = m.get("gpu__time_duration.sum", 0.0)
    a = agg[names[i][:80]]
    a[0] += 1
    a[1] += b
    a[2] += t
    tb += b
    tt += t
print(f"{'kernel':82s} {'launches':>8s} {'GB':>9s} {'ms':>9s} {'GB/s':>8s} {'time%':>6s}")
for n, (c, b, t) in sorted(agg.items(), key=lambda x: -x[1][2]):
    print(f"{n:82s} {c:8d} {b / 1e9:9.3f} {t * 1e3:9.3f} {b / t / 1e9 if t else 0:8.0f} {100 * t / tt:6.1f}")
g = open(sys.argv[2]).read() if len(sys.argv) > 2 else ""
m = re.search(r"iterations (\d+) .* ms ([0-9.]+)", g)
its, step_ms = (int(m.group(1)), float(m.group(2))) if m else (None, None)
print(f"step: {len(launch)} launches, {tb / 1e9:.3f} GB DRAM, {tt * 1e3:.3f} ms summed kernel time "
      f"(serialised under ncu) = {tb / tt / 1e9:.0f} GB/s")
rec = {"workload": sys.argv[3] if len(sys.argv) > 3 else None, "launches": len(launch),
       "dram_bytes_per_step": tb, "kernel_ms_serialised": tt * 1e3, "iterations": its,
       "step_ms_graph": step_ms,
       "dram_bytes_per_iteration": tb / its if its else None,
       "achieved_gbs_in_step": tb / (step_ms * 1e-3) / 1e9 if step_ms else None}
if step_ms:
    print(f"graph-mode step {step_ms:.3f} ms ({its} iterations): {rec['achieved_gbs_in_step']:.0f} GB/s of measured DRAM traffic")
print(json.dumps(rec))
