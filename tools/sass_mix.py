"""Opcode mix and stall samples per opcode from an ncu source-page CSV (SASS view).
usage: python tools/sass_mix.py gpurun_out/ncu_<k>_<skip>_src.csv.gz [top]"""
import csv
import gzip
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(gzip.open(path, "rt")))
h = rows[1]
iS, iX = h.index("Source"), h.index("Instructions Executed")
iW = h.index("Warp Stall Sampling (All Samples)")
ex, st = defaultdict(float), defaultdict(float)
for r in rows[2:]:
    if len(r) <= iX:
        continue
    s = r[iS].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1]
    op = s.split()[0] if s else "?"
    op = op.split(".")[0]
    ex[op] += float(r[iX] or 0)
    st[op] += float(r[iW] or 0)
tx, ts = sum(ex.values()), sum(st.values())
print(f"instructions {tx:.0f}, stall samples {ts:.0f}")
for op in sorted(ex, key=lambda o: -ex[o])[:top]:
    print(f"{op:10s} inst {100*ex[op]/tx:5.1f}%   samples {100*st[op]/ts:5.1f}%")
