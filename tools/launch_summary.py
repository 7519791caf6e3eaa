"""Summarise an ncu --csv launch list (gpu__time_duration.sum): time per kernel name and grid."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
gi = h.index("Grid Size") if "Grid Size" in h else None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][-48:] + (" g=" + r[gi] if gi is not None else "")
    v = float(r[vi].replace(",", ""))
    v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(r[ui], v)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print(f"total {tot / 1e3:.2f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{k:72s} {n:5d} {t / 1e3:9.3f} ms {100 * t / tot:5.1f}%")
