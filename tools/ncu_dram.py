"""DRAM bytes and duration per launch of an ncu --set full report: python tools/ncu_dram.py rep [iters]
(prints dram read+write bytes, gpu__time_duration and, with iters, the per-iteration DRAM bytes)."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))

    def val(k):
        v = float(d[k].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                    "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(u[k], 1.0)

    rd, wr, dur = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
    print(f"{d['Kernel Name'][:90]}: dram read {rd / 1e6:.1f} MB write {wr / 1e6:.1f} MB, {dur * 1e3:.3f} ms, "
          f"{(rd + wr) / dur / 1e9:.0f} GB/s, regs {d.get('launch__registers_per_thread')}")
    if len(sys.argv) > 2:
        print(f"  per iteration: {(rd + wr) / int(sys.argv[2]):.0f} bytes")
