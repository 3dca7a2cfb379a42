"""Summarise gpurun_out/prof_<tag>_* (ncu) into profiles/<tag>_*.txt for the commit.

  python tools/summarize_profiles.py r01
"""
import collections
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
SRC = os.path.join(ROOT, "gpurun_out")
DST = os.environ.get("PROFILE_DST") or os.path.join(ROOT, "profiles")
PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data:
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    lines = [f"{'us':>10} {'share':>6} {'n':>5} {'avg us':>9}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t:10.1f} {100 * t / tot:5.1f}% {n:5d} {t / n:9.1f}  {k}")
    lines.append(f"total {tot:.1f} us over {len(data)} launches")
    return "\n".join(lines)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return "(empty)"
    h = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "?").split("(")[0]
        dur_us = float(d.get("gpu__time_duration.sum", "0").replace(",", "")) / 1e3 if d.get(
            "gpu__time_duration.sum") else 0.0
        unit = "usecond"
        out.append(f"kernel {name}")
        for m in METRICS:
            if m in d:
                out.append(f"  {m:70s} {d[m]}")
        rb = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
        wb = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
        out.append(f"  dram traffic read+write (ncu units as above)          {rb + wb:.3f}")
    return "\n".join(out)


os.makedirs(DST, exist_ok=True)
lp = os.path.join(SRC, f"prof_{TAG}_launches.csv")
if os.path.exists(lp):
    hdr = ("# ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 400 "
           "python bench.py --steps 1 --warmup 1 --no-cpu\n"
           "# cold-cache, serialised launches: compare shares, not absolutes\n")
    open(os.path.join(DST, f"{TAG}_launches_summary.txt"), "w").write(hdr + launches(lp) + "\n")
for rep in sorted(glob.glob(os.path.join(SRC, f"prof_{TAG}_*.ncu-rep"))):
    name = os.path.basename(rep)[len(f"prof_{TAG}_"):-len(".ncu-rep")]
    body = full(rep)
    hdr = f"# ncu --set full --clock-control none capture ({name}); peaks: {PEAKS.get('hbm_gbs')} GB/s, {PEAKS.get('bf16_tflops')} TFLOP/s measured\n"
    open(os.path.join(DST, f"{TAG}_ncu_{name}.txt"), "w").write(hdr + body + "\n")
print(sorted(os.listdir(DST)))
