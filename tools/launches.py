"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0].replace("void ", "")[:60]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for k, v in agg.items() if "sfcb200" in k)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = f"{100*sum(v)/tot:5.1f}%" if "sfcb200" in k else "  -  "
    print(f"{k:62s} n={len(v):3d} mean_us={sum(v)/len(v)/1e3:9.2f} total_us={sum(v)/1e3:10.1f} {share}")
