"""Per-source-line warp-stall summary of an ncu report (--import-source, -lineinfo build):
python tools/ncu_lines.py report.ncu-rep [top]   (runs ncu -i ... --print-source cuda,sass)."""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
reasons = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
wi = h.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[hi + 1:]:
    if len(r) > wi and r[0] and r[2] == "-":
        try:
            w = int(r[wi])
        except ValueError:
            continue
        rs = collections.Counter({h[i][6:]: int(r[i] or 0) for i in reasons})
        lines.append((w, int(r[0]), r[1].strip()[:80], rs))
tot = sum(x[0] for x in lines)
allr = collections.Counter()
for x in lines:
    allr.update(x[3])
print("total samples", tot, " by reason:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in allr.most_common(8)))
for w, l, src, rs in sorted(lines, key=lambda x: -x[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = ", ".join(f"{k} {100 * v / max(w, 1):.0f}%" for k, v in rs.most_common(3) if v)
    print(f"{w:7d} {100 * w / tot:5.1f}% L{l:4d} {src:80s} [{top}]")
