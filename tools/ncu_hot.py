"""Hot SASS lines of one kernel from `ncu -i rep --page source --csv --print-source sass -k regex:NAME`:
prints total executed instructions, stall-sample totals and the top lines by samples."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
sel = ["--launch-skip", kern, "--launch-count", "1"] if kern.isdigit() else ["-k", f"regex:{kern}"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", *sel, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
data = []
for r in rows[hi + 1:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(h):
        data.append(r)
c = {k: h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed")}
num = lambda s: float(s.replace(",", "") or 0)
tot_i = sum(num(r[c["Instructions Executed"]]) for r in data)
tot_s = sum(num(r[c["Warp Stall Sampling (All Samples)"]]) for r in data)
print(f"warp-instructions executed {tot_i:.0f}   stall samples {tot_s:.0f}")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(num(r[h.index(k)]) for r in data) for k in stalls}
print("stalls:", ", ".join(f"{k[6:]}={v:.0f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for r in sorted(data, key=lambda r: -num(r[c["Warp Stall Sampling (All Samples)"]]))[:top]:
    print(f"{r[c['Address']]:>8s} {num(r[c['Warp Stall Sampling (All Samples)']]):6.0f} {num(r[c['Instructions Executed']]):8.0f}  {r[c['Source']][:90]}")
