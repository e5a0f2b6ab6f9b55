"""Turn a round's profile captures (tools/capture_profiles.sh -> gpurun_out/prof) into the
tracked summaries under profiles/:

  profiles/rNN_launches_w2.txt   per-kernel share of the default bench command's launches
  profiles/rNN_ncu_w{2,5}.txt    ncu --set full key counters per stage kernel and variant
  profiles/ncu_traffic.json      dram read+write bytes per launch, averaged over variants,
                                 keyed "<workload name>:<stage>" (read by bench.py)

    python tools/make_profile_summaries.py r01
"""
import collections, csv, json, os, re, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_02913_b200 import workloads as wl  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out", "prof")
dst = os.path.join(ROOT, "profiles")
VARIANTS = ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3"]


def stage_of(name):
    if "k_act_row<" in name:  # register-resident SWAR transform: MODE 0/2 absmax (+kept V), 1 quantize
        return "quantize" if re.search(r"k_act_row<\d+, 1,", name) else "absmax"
    if "k_act_pair<" in name:  # the two-channel SWAR form (large layers)
        return "absmax" if re.search(r"k_act_pair<\d+, 0>", name) else "act_quant"
    if "k_act<" in name:
        return "absmax" if re.search(r"k_act<\d+, 0,", name) else "act_quant"
    for key, st in (("k_quant_kept", "quantize"), ("k_gemm", "gemm"), ("k_output", "output"),
                    ("k_zero_words", "reset")):
        if key in name:
            return st
    return None


# ---------------------------------------------------------------- launch list
rows = list(csv.reader(l for l in open(os.path.join(src, "launches_w2.csv")) if l.startswith('"')))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    k = re.sub(r"\(.*", "", r[ik]).replace("sfcb200::", "").replace("void ", "")
    k = re.sub(r"<(\d+), (\d+), \d+>", r"<\1, \2, CC>", k)
    tot[k] += float(r[iv]) / 1e3
    cnt[k] += 1
ours = {k: v for k, v in tot.items() if k.split("<")[0] in ("k_zero_words", "k_act", "k_act_row", "k_act_pair",
                                                           "k_quant_kept", "k_gemm", "k_output", "k_output_pers",
                                                           "k_output_smallc", "k_output_reg")}
s_all = sum(ours.values())
with open(os.path.join(dst, f"{tag}_launches_w2.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none of\n"
            "#   python bench.py --steps 2 --warmup 3 --no-cpu-baseline      (workload 2, default)\n"
            "# cold-cache, serialised per-launch times (the bench's own events time the chained step);\n"
            "# shares are over the per-call kernels of every launch in the run (warm-up, timed, e2e,\n"
            "# per-stage timing).\n")
    f.write(f"{'kernel':36s} {'launches':>8s} {'total us':>10s} {'avg us':>8s} {'share':>6s}\n")
    for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
        f.write(f"{k:36s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:8.2f} {100 * v / s_all:5.1f}%\n")
    other = {k: v for k, v in tot.items() if k not in ours}
    f.write(f"\nother launches in the run (setup, torch, L2 flush): " +
            ", ".join(f"{k} x{cnt[k]}" for k in sorted(other)) + "\n")

# ---------------------------------------------------------------- full captures
WANT = [("gpu__time_duration.sum", "us", 1.0), ("dram__bytes_read.sum", "MB", None), ("dram__bytes_write.sum", "MB", None),
        ("lts__t_sectors.sum", "sectors", 32e-6), ("inst_executed.sum", "Minst", 1e-6),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%", 1.0),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "%", 1.0),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "%", 1.0),
        ("launch__grid_size", "", 1.0), ("launch__registers_per_thread", "", 1.0)]


def to_base(val, unit):
    try:
        v = float(val.replace(",", ""))
    except ValueError:
        return float("nan")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "nsecond": 1e-3, "ns": 1e-3,
             "msecond": 1e3, "ms": 1e3}
    return v * scale.get(unit, 1)


traffic = collections.defaultdict(list)
for w in (2, 5):
    name = wl.WORKLOADS[w].name
    lines = [f"# ncu --set full --clock-control none, second forward of tools/prof_once.py --workload {w}\n"
             f"# ({name}); one launch per stage kernel and variant.  dram = HBM bytes of that launch.\n"]
    hdr = f"{'variant':13s} {'stage':9s} {'us':>8s} {'dramR MB':>9s} {'dramW MB':>9s} {'L2 MB':>8s} {'Minst':>7s} " \
          f"{'issue%':>7s} {'warps%':>7s} {'tensor%':>8s} {'grid':>6s} {'regs':>5s}\n"
    lines.append(hdr)
    for v in VARIANTS:
        p = os.path.join(src, f"full_w{w}_{v}.raw.csv")
        if not os.path.exists(p):
            continue
        rr = list(csv.reader(open(p)))
        h, units, data = rr[0], rr[1], rr[2:]
        for d in data:
            st = stage_of(d[h.index("Kernel Name")])
            if st is None:
                continue
            vals = []
            for m, u, sc in WANT:
                cands = [j for j, k in enumerate(h) if k == m] or \
                        [j for j, k in enumerate(h) if k.endswith(m) and k.split(".")[0] in ("sm__inst_executed", "smsp__inst_executed")] or \
                        [j for j, k in enumerate(h) if k.endswith("." + m)]
                if not cands:
                    vals.append(float("nan"))
                    continue
                i = cands[0]
                if u == "MB":
                    vals.append(to_base(d[i], units[i]) / 1e6)
                elif u == "us":
                    vals.append(to_base(d[i], units[i]))
                else:
                    try:
                        vals.append(float(d[i].replace(",", "")) * sc)
                    except ValueError:
                        vals.append(float("nan"))
            dram = (vals[1] + vals[2]) * 1e6
            traffic[f"{name}:{st}"].append(dram)
            lines.append(f"{v:13s} {st:9s} {vals[0]:8.1f} {vals[1]:9.2f} {vals[2]:9.2f} {vals[3]:8.1f} {vals[4]:7.2f} "
                         f"{vals[5]:7.1f} {vals[6]:7.1f} {vals[7]:8.1f} {vals[8]:6.0f} {vals[9]:5.0f}\n")
    with open(os.path.join(dst, f"{tag}_ncu_w{w}.txt"), "w") as f:
        f.writelines(lines)
out = {k: sum(v) / len(v) for k, v in sorted(traffic.items())}
out["_note"] = (f"{tag}: dram__bytes_read.sum + dram__bytes_write.sum per launch from ncu --set full "
                "(cold caches), averaged over the three variants; tools/make_profile_summaries.py")
with open(os.path.join(dst, "ncu_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(open(os.path.join(dst, f"{tag}_launches_w2.txt")).read())
print(open(os.path.join(dst, f"{tag}_ncu_w2.txt")).read())
print(open(os.path.join(dst, f"{tag}_ncu_w5.txt")).read())
