"""Attribute an ncu SASS profile to kernel source lines (outermost inline frame).

    python tools/sass_lines.py REP LAUNCH_INDEX OBJ.o FUNC_REGEX [TOP]

REP: .ncu-rep captured with -lineinfo builds; LAUNCH_INDEX: index of the launch in REP;
OBJ.o: the object file holding the kernel (the same build that was profiled);
FUNC_REGEX: regex matching the mangled kernel name in that object.
Prints warp-instructions executed and stall samples per source line, largest first.
"""
import collections, csv, os, re, subprocess, sys, tempfile

rep, idx, obj, fre = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", idx, "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
num = lambda s: float(s.replace(",", "") or 0)
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[h.index("Address")].startswith("0x")]
ca, ci, cs = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = min(int(r[ca], 16) for r in data)

with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
loc, cur, in_fn = {}, None, False
for line in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        in_fn = re.search(fre, m.group(1)) is not None
        continue
    if not in_fn:
        continue
    if line.lstrip().startswith("//## File"):
        frames = re.findall(r'"([^"]+)", line (\d+)', line)
        f, l = frames[-1]
        cur = (os.path.basename(f), int(l))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        loc[int(m.group(1), 16)] = cur
agg_i, agg_s = collections.Counter(), collections.Counter()
for r in data:
    k = loc.get(int(r[ca], 16) - base, ("?", 0))
    agg_i[k] += num(r[ci])
    agg_s[k] += num(r[cs])
src = {}
def text(k):
    f, l = k
    for root in ("paper_2407_02913_b200/csrc",):
        p = os.path.join(root, f)
        if os.path.exists(p):
            if p not in src:
                src[p] = open(p).read().splitlines()
            return src[p][l - 1].strip()[:80] if 0 < l <= len(src[p]) else ""
    return ""
ti, ts = sum(agg_i.values()), sum(agg_s.values())
print(f"{len(loc)} SASS offsets mapped; warp-instr {ti:.0f}, stall samples {ts:.0f}")
for k, v in sorted(agg_i.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{k[0]:>16s}:{k[1]:<4d} instr {100 * v / ti:5.1f}%  stalls {100 * agg_s[k] / max(ts, 1):5.1f}%  {text(k)}")
