"""Per-launch summary of an ncu --csv launch list (time, DRAM read/write, achieved GB/s).

    python tools/launch_summary.py gpurun_out/r2/launch_w4.csv [--min-us 5]
"""
import argparse, collections, csv, io

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--min-us", type=float, default=0.0)
a = ap.parse_args()
txt = open(a.csv).read()
txt = txt[txt.index('"ID"'):]
k = collections.OrderedDict()
for r in csv.DictReader(io.StringIO(txt)):
    name = r["Kernel Name"]
    short = name.split("(")[0]
    k.setdefault((r["ID"], short, r["Grid Size"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tot = collections.Counter()
for (i, n, g), m in k.items():
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    rd, wr = m.get("dram__bytes_read.sum", 0) / 1e6, m.get("dram__bytes_write.sum", 0) / 1e6
    base = n.split("<")[0]
    tot[base] += t
    if t >= a.min_us:
        print(f"{i:>4} {n[:48]:48s} {g:16s} {t:9.1f}us R {rd:8.1f}MB W {wr:8.1f}MB {(rd + wr) / max(t, 1e-9) / 1e3:6.2f}TB/s")
print("totals (us):", {k_: round(v, 1) for k_, v in tot.most_common()})
