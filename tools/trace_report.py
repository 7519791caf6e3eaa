"""Summarise a KPP_TRACE dump: per-iteration critical path across CTAs (ns, globaltimer)."""
import sys
import numpy as np
d = np.fromfile(sys.argv[1], dtype=np.int64)
T, G = int(d[0]), int(d[1])
tr = d[2:].reshape(T, G, 8).astype(np.float64)
names = ["start", "P1 done", "partials in", "cl.partial out", "gather done", "r done", "y done", "end"]
for t in range(1, T):
    base = tr[t, :, 0].min()
    x = tr[t] - base
    row = []
    for e in range(8):
        v = x[:, e]
        row.append(f"{names[e]}: min {v.min():6.0f} med {np.median(v):6.0f} max {v.max():6.0f}")
    if t < 4:
        print(f"iter {t}:\n  " + "\n  ".join(row))
# averages over iterations of the median and max per event
mx = np.array([[ (tr[t,:,e]-tr[t,:,0].min()).max() for e in range(8)] for t in range(1,T)])
md = np.array([[ np.median(tr[t,:,e]-tr[t,:,0].min()) for e in range(8)] for t in range(1,T)])
print("mean over iterations (ns since earliest start):")
for e in range(8):
    print(f"  {names[e]:16s} median {md[:,e].mean():7.0f}   max {mx[:,e].mean():7.0f}")
per = np.diff(tr[:,:,0].min(axis=1))
print("iteration period (ns):", per.mean())
