"""Summarise an ncu --page source --csv --print-source sass export: stall reasons summed over
instruction groups (by execution count) and the hottest lines.
  python tools/ncu_lines.py export.csv [top]"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
groups = collections.defaultdict(lambda: collections.Counter())
lines = []
for r in rows[2:]:
    try:
        e = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    g = groups[e]
    g["_lines"] += 1
    g["_samples"] += s
    for k in stall_cols:
        try:
            g[k] += int(r[ix[k]] or 0)
        except ValueError:
            pass
    lines.append((s, r[ix["Address"]][-5:], e, r[ix["Source"]][:80],
                  {k: r[ix[k]] for k in stall_cols if r[ix[k]] not in ("", "0")}))
tot = sum(g["_samples"] for g in groups.values())
print(f"total samples {tot}")
for e, g in sorted(groups.items(), key=lambda kv: -kv[1]["_samples"])[:12]:
    st = ", ".join(f"{k[6:]}={v}" for k, v in g.most_common() if not k.startswith("_") and v > 0)
    print(f"exec {e:9d} lines {g['_lines']:5d} samples {g['_samples']:6d}: {st}")
lines.sort(reverse=True)
for s, a, e, src, st in lines[:top]:
    print(f"{s:6d} {a} {e:9d} {src:60s} {st}")
