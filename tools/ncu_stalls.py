"""Top warp-stall sample sites of an .ncu-rep (source page, SASS) with the preceding
instructions, and the barrier-wait attribution: python tools/ncu_stalls.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
h, data = rows[hi], rows[hi + 1:]
si, src, ad = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Address")
data = [r for r in data if len(r) > si]
tot = sum(float(r[si] or 0) for r in data) or 1.0
idx = {r[ad]: i for i, r in enumerate(data)}
print(f"{rep}: {tot:.0f} warp-stall samples")
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
    i = idx[r[ad]]
    ctx = " | ".join(x[src].strip()[:48] for x in data[max(0, i - 2):i])
    print(f"{float(r[si]):7.0f} {100 * float(r[si]) / tot:5.1f}%  {r[src].strip()[:46]:46s} <- {ctx}")
