"""Per-position kernel times of one GMRES iteration from an ncu launch list
(host-driven mode): averages iterations 5..24 between k_dgs_update launches."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[h]
ki, gi, vi = H.index("Kernel Name"), H.index("Grid Size"), H.index("Metric Value")
L = [(r[ki].split("(")[0].replace("void unnamed>::", "").replace("unnamed>::", ""), r[gi],
      float(r[vi].replace(",", ""))) for r in rows[h + 1:] if len(r) > vi]
ups = [i for i, x in enumerate(L) if x[0].startswith("k_dgs_update")]
seqs = [L[ups[k] + 1:ups[k + 1] + 1] for k in range(5, min(25, len(ups) - 1))]
n = len(seqs[0])
tot = 0.0
for q in range(n):
    t = sum(s[q][2] for s in seqs) / len(seqs)
    tot += t
    print(f"{q:3d} {seqs[0][q][0]:38s} {seqs[0][q][1]:>14s} {t / 1000:7.2f} us")
print(f"iteration total {tot / 1000:.1f} us over {len(seqs)} iterations")
