"""Hot SASS lines and opcode mix of an `ncu --page source --csv` export."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iI = h.index("Instructions Executed"); iSrc = h.index("Source")
iN = h.index("Warp Stall Sampling (Not-issued Samples)")
print("total samples", sum(int(r[iS] or 0) for r in data), "total warp inst", sum(int(r[iI] or 0) for r in data))
for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{int(r[iS]):7d} {int(r[iN]):7d} {int(r[iI]):10d}  {r[0][-5:]} {r[iSrc].strip()[:90]}")
c = Counter()
for r in data:
    op = r[iSrc].strip().split()
    if op:
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += int(r[iI] or 0)
print(c.most_common(22))
