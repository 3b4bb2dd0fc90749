"""Key metrics of ncu --set full captures (.ncu-rep) as a text table."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp_inst"),
]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if not rows:
        continue
    h, units = rows[0], rows[1]
    print(f"== {rep}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        cols = []
        for k, short in KEYS:
            if k in h:
                i = h.index(k)
                cols.append(f"{short}={r[i]}{units[i] if units[i] not in ('', 'inst') else ''}")
        print(f"  {name[:60]:60s} " + " ".join(cols))
