"""Executed warp-instructions and stall samples per CUDA source line of one kernel launch
(ncu --page source --print-source cuda,sass):
    python tools/ncu_lines.py REP LAUNCH_INDEX [TOP]"""
import csv, subprocess, sys
from collections import defaultdict
rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", k, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
num = lambda s: float(s.replace(",", "")) if s.replace(",", "").replace(".", "", 1).isdigit() else 0.0
hdr, fname, line, src = None, "", 0, ""
ins, st, text = defaultdict(float), defaultdict(float), {}
for r in csv.reader(raw.splitlines()):
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        line, src = int(r[0]), r[1]
        text[(fname, line)] = src.strip()[:90]
    if r[2]:  # a SASS row under the current source line
        ins[(fname, line)] += num(r[hdr.index("Instructions Executed")])
        st[(fname, line)] += num(r[hdr.index("Warp Stall Sampling (All Samples)")])
tot = sum(ins.values()) or 1
print(f"total warp-instructions {tot:.0f}, stall samples {sum(st.values()):.0f}")
for key in sorted(ins, key=lambda q: -ins[q])[:top]:
    print(f"{key[0][:14]:14s}{key[1]:5d} {ins[key]:10.0f} {100*ins[key]/tot:5.1f}% {st[key]:6.0f}  {text.get(key, '')}")
