"""Summarise an ncu --csv launch list (gpu__time_duration.sum) of tools/launch_list.py into a
per-kernel-name table and an ordered per-launch list.  python tools/launch_table.py file.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
gi = h.index("Grid Size") if "Grid Size" in h else None
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
seq = []
for r in data:
    v = float(r[vi].replace(",", "")) / 1e3  # ns -> us
    name = r[ki].split("(")[0][:90]
    agg[name][0] += 1; agg[name][1] += v; tot += v
    seq.append((r[ii], name, v, r[gi] if gi is not None else ""))
print(f"total {tot:.1f} us over {len(seq)} launches")
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v:10.1f} us {100*v/tot:5.1f}% n={n:4d} avg {v/n:8.1f}  {k}")
if "-v" in sys.argv:
    for i, n, v, g in seq:
        print(f"{i:>5} {v:9.1f} {g:>16} {n}")
