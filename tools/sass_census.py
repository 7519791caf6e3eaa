"""Per-kernel SASS census of libkpp.so (cuobjdump -sass): counts of the instructions that show
which hardware paths a kernel uses -- DMMA (FP64 tensor core, mma.sync.m8n8k4.f64), UTMALDG (TMA
tensor loads incl. tile::gather4), UBLKCP (TMA bulk copies), STAS (st.async DSMEM stores), SYNCS
(mbarrier operations), LDGSTS (cp.async), UTC*MMA / LDTM (tcgen05; none expected: no f64 kind),
DFMA (FP64 FMA pipe), plus the instruction total.  Usage: python tools/sass_census.py [lib] > out"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2501_11673_b200/libkpp.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["DMMA", "DFMA", "UTMALDG", "UBLKCP", "STAS", "SYNCS", "LDGSTS", "UTCHMMA|UTCQMMA|UTCIMMA|UTCMMA", "LDTM",
        "HMMA", "BAR", "SHFL"]
cnt = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        cnt[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if not m:
        continue
    op = m.group(2).split(".")[0]
    cnt[cur]["total"] += 1
    for k in KEYS:
        if re.fullmatch(k, op):
            cnt[cur][k.split("|")[0] if "|" not in k else "UTC*MMA"] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else names


names = list(cnt)
dn = demangle(names)
cols = ["DMMA", "DFMA", "UTMALDG", "UBLKCP", "STAS", "SYNCS", "LDGSTS", "UTC*MMA", "LDTM", "HMMA", "BAR", "SHFL", "total"]
print("# SASS census of", lib, "(cuobjdump -sass; per kernel; sm_100a)")
print("kernel\t" + "\t".join(cols))
tot = collections.Counter()
for n, d in sorted(zip(names, dn), key=lambda z: z[1]):
    c = cnt[n]
    tot.update(c)
    short = re.sub(r"\(.*", "", d.replace("(anonymous namespace)::", ""))[:110]
    print(short + "\t" + "\t".join(str(c.get(k, 0)) for k in cols))
print("ALL\t" + "\t".join(str(tot.get(k, 0)) for k in cols))
