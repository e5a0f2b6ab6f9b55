"""Round-2 profile summaries (tools/capture_r02.sh -> gpurun_out/prof) into profiles/:

  r02_bench_w4.json      the default bench line of the capture run (config 4)
  r02_launches_w4.txt    per-kernel totals / shares of the ncu launch list of the default bench
  r02_layers_w4.txt      per layer and kernel of one config-4 forward: time, HBM read / write
  r02_layers_w5.txt      the same for config 5
  r02_ncu_full.txt       --set full counters of the stage kernels (VGG-16 layers 1 and 8, config 5)
  ncu_traffic.json       HBM bytes of one forward per workload ("<workload>:step"), read by bench.py

    python tools/summarize_r02.py
"""
import collections, csv, json, os, re, shutil, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")
TAG = "r02"


def kname(s):
    s = re.sub(r"\(.*", "", s).replace("sfcb200::", "").replace("void ", "").replace("(anonymous namespace)::", "")
    return s.replace("<unnamed>::", "").strip()


def ncu_rows(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    return rows[0], rows[1:]


def launch_list():
    h, rows = ncu_rows(os.path.join(SRC, "launches_w4.csv"))
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        v = float(r[iv].replace(",", ""))
        v = v / 1e3 if r[iu] in ("ns", "nsecond") else (v * 1e3 if r[iu] in ("ms", "msecond") else v)  # -> us
        k = kname(r[ik])
        tot[k] += v
        cnt[k] += 1
    s_all = sum(tot.values())
    out = ["# ncu --metrics gpu__time_duration.sum --clock-control none of",
           "#   python bench.py --steps 2 --warmup 3 --no-cpu-baseline      (config 4, the default line)",
           "# cold-cache, serialised per-launch times of every launch in the run (warm-up, timed, e2e,",
           "# per-stage timing); compare kernel SHARES with the bench's event timing, not absolutes.",
           f"{'kernel':44s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"{k[:44]:44s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:9.2f} {100 * v / s_all:5.1f}%")
    return "\n".join(out) + "\n"


def layers(wl):
    h, rows = ncu_rows(os.path.join(SRC, f"layers_w{wl}.csv"))
    ik, iid, im, iv, iu = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.OrderedDict()
    for r in rows:
        key = (int(r[iid]), kname(r[ik]))
        v = float(r[iv].replace(",", ""))
        u = r[iu]
        if r[im] == "gpu__time_duration.sum":
            v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        else:
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        per.setdefault(key, {})[r[im]] = v
    out = [f"# one forward of each layer of workload {wl} (tools/layer_launches.py), ncu per launch:",
           "# time (cold caches), HBM bytes read / written.  One-time kernels (filter transform, quantizer",
           "# table) are listed but are not part of the per-call step.",
           f"{'id':>4s} {'kernel':44s} {'us':>9s} {'read MB':>9s} {'write MB':>9s}"]
    step = 0.0
    layer_ix = -1
    for (i, k), m in per.items():
        if k.startswith("k_filter_prepare"):
            layer_ix += 1
            out.append(f"---- layer {layer_ix}")
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        out.append(f"{i:4d} {k[:44]:44s} {m.get('gpu__time_duration.sum', 0):9.1f} {rd / 1e6:9.1f} {wr / 1e6:9.1f}")
        if not (k.startswith("k_filter_prepare") or k.startswith("k_build_qtable")):
            step += rd + wr
    out.append(f"# per-call HBM traffic of one step (all layers): {step / 1e9:.3f} GB")
    return "\n".join(out) + "\n", step


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread"]


def full(tag):
    path = os.path.join(SRC, f"full_{tag}.raw.csv")
    if not os.path.exists(path):
        return f"# {tag}: capture missing\n"
    rows = list(csv.reader(open(path)))
    h, u, data = rows[0], rows[1], rows[2:]
    ix = {w: h.index(w) for w in WANT if w in h}
    out = [f"# {tag}"]
    for r in data:
        out.append("  " + kname(r[h.index("Kernel Name")])[:70])
        for w, i in ix.items():
            out.append(f"      {w:68s} {r[i]:>14s} {u[i]}")
    return "\n".join(out) + "\n"


def main():
    os.makedirs(DST, exist_ok=True)
    b = os.path.join(SRC, "bench_default.json")
    if os.path.exists(b):
        line = open(b).read().strip().splitlines()[-1]
        json.loads(line)
        open(os.path.join(DST, f"{TAG}_bench_w4.json"), "w").write(line + "\n")
    open(os.path.join(DST, f"{TAG}_launches_w4.txt"), "w").write(launch_list())
    traffic = {}
    for wl, name in ((4, "cfg4_vgg16_b128"), (5, "cfg5_n256_c512_14")):
        txt, step = layers(wl)
        open(os.path.join(DST, f"{TAG}_layers_w{wl}.txt"), "w").write(txt)
        traffic[f"{name}:step"] = step
    traffic["_note"] = ("r02: dram__bytes_read.sum + dram__bytes_write.sum summed over the per-call kernels of one "
                        "forward of every layer (ncu per launch, cold caches; tools/summarize_r02.py)")
    json.dump(traffic, open(os.path.join(DST, "ncu_traffic.json"), "w"), indent=1)
    with open(os.path.join(DST, f"{TAG}_ncu_full.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none, second forward of tools/prof_once.py (int8 requant\n"
                "# outputs for VGG-16, int32 y + fp32 for config 5): one launch per stage kernel.\n")
        for t in ("w4_l1", "w4_l8", "w5_l0"):
            f.write(full(t))
    print("wrote", sorted(p for p in os.listdir(DST) if p.startswith(TAG)))


if __name__ == "__main__":
    main()
