"""Generate the committed golden fixtures from the *reference itself* (oracle/_ref, built
from /root/reference/proj/src by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py            (qconv_cases.npz, catalog_3x3.json)
    python tests/golden/make_golden.py --large-r  (qconv_large_r.npz, catalog_large_r.json)
    python tests/golden/make_golden.py --real     (qconv_real.npz)
    python tests/golden/make_golden.py --cli      (cli_golden.json, cli_layers.json)

Writes tests/golden/catalog_3x3.json (the reference's catalog export restricted to the
three 3x3 SFC specs + the full-catalog FNV hash) and tests/golden/qconv_cases.npz (seeded
int8 inputs, the reference's quantized_fast_conv2d output and report, its fp64
direct_conv2d and transform_filters, and scalar known answers).  The fixtures pin the
oracle and the GPU path on a box where /root/reference does not exist.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bindings as ob  # noqa: E402

VARIANTS = ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3"]
LARGE_R = ["sfc6-6x6-5x5", "sfc6-4x4-7x7"]  # catalog.cpp:249-250

# (tag, B, C, OC, H, W, pad, lo, bits) for the 5x5 / 7x7 variants (their own RNG and file)
LARGE_CASES = [
    ("small_p2", 1, 6, 5, 15, 15, 2, -128, 8),
    ("ragged_p3", 2, 3, 4, 13, 11, 3, -128, 8),
    ("relu_p1", 1, 9, 3, 12, 12, 1, 0, 8),
    ("bits4_p0", 1, 4, 3, 14, 14, 0, -128, 4),
    ("tiny", 1, 2, 2, 7, 7, 3, -128, 8),
]

# (tag, B, C, OC, H, W, pad, lo, bits, act_scope, filter_scope, search)
CASES = [
    ("small_p1", 1, 8, 8, 14, 14, 1, -128, 8, 0, 0, 0),
    ("ragged_p1", 2, 5, 3, 13, 11, 1, -128, 8, 0, 0, 0),
    ("relu_p0", 1, 16, 4, 12, 12, 0, 0, 8, 0, 0, 0),
    ("pad2", 1, 4, 6, 9, 10, 2, -128, 8, 0, 0, 0),
    ("bits4", 1, 6, 5, 11, 11, 1, -128, 4, 0, 0, 0),
    ("bits6", 1, 6, 5, 11, 11, 1, -128, 6, 0, 0, 0),
    ("bits2", 1, 3, 2, 8, 8, 1, -128, 2, 0, 0, 0),
    ("bits12", 1, 3, 2, 8, 8, 1, -128, 12, 0, 0, 0),
    ("actfreq", 1, 6, 4, 12, 12, 1, -128, 8, 1, 0, 0),
    ("filfreq", 1, 6, 4, 12, 12, 1, -128, 8, 0, 1, 0),
    ("filchfreq", 1, 6, 4, 12, 12, 1, -128, 8, 1, 2, 0),
    ("msegrid", 1, 3, 3, 10, 10, 1, -128, 8, 0, 0, 1),
    ("tiny_h", 1, 2, 2, 3, 3, 1, -128, 8, 0, 0, 0),
]


def exact_texts(js, names):
    """The exact substring of the reference's catalog export for each algorithm."""
    full = json.loads(js)
    sel = [a for a in full["algorithms"] if a["name"] in names]
    exact = {}
    for a in sel:
        tail = js[js.index('{"name":"' + a["name"]):]
        depth = 0
        for i, ch in enumerate(tail):
            depth += ch == "{"
            depth -= ch == "}"
            if depth == 0:
                exact[a["name"]] = tail[: i + 1]
                break
    return sel, exact


def large_r():
    """tests/golden/catalog_large_r.json + qconv_large_r.npz for the 5x5 / 7x7 variants."""
    js, h = ob.ref_catalog_json()
    sel, exact = exact_texts(js, LARGE_R)
    with open(os.path.join(HERE, "catalog_large_r.json"), "w") as f:
        json.dump({"full_catalog_fnv1a64": f"{h:016x}", "algorithms": sel, "exact_text": exact}, f, indent=1)
    arrays = {}
    rng = np.random.default_rng(0x5FC1)
    for tag, B, C, OC, H, W, pad, lo, bits in LARGE_CASES:
        x = rng.integers(lo, 128, size=(B, C, H, W), dtype=np.int8)
        arrays[f"{tag}/x"] = x
        arrays[f"{tag}/meta"] = np.array([pad, bits], np.int64)
        for v in LARGE_R:
            R = ob.spec(v, source="ref")["R"]
            w = rng.integers(-127, 128, size=(OC, C, R, R), dtype=np.int8)
            arrays[f"{tag}/{v}/w"] = w
            arrays[f"{tag}/{v}/direct"] = ob.ref_direct_conv2d(x, w, pad)
            out, rep = ob.ref_quantized_fast_conv2d(x, w, v, pad, bits)
            arrays[f"{tag}/{v}/out"] = out
            arrays[f"{tag}/{v}/report"] = np.array([rep["mse"], rep["signal_energy"], rep["snr_db"],
                                                    rep["saturations"], rep["values_quantized"]], np.float64)
            if tag == "small_p2":
                arrays[f"{tag}/{v}/u"] = ob.ref_transform_filters(w, v)
    np.savez_compressed(os.path.join(HERE, "qconv_large_r.npz"), **arrays)
    print("wrote", len(arrays), "large-R arrays")


# (tag, B, C, OC, H, W, act_scope, filter_scope, search, bits) with real-valued N(0, 1)
# inputs and filters, the values the reference CLI's quantsim feeds (sfconv_cli.cpp:299-300)
REAL_CASES = [
    ("real_default", 1, 5, 4, 12, 12, 0, 0, 0, 8),
    ("real_actfreq", 2, 3, 3, 10, 11, 1, 0, 0, 8),
    ("real_chfreq_mse", 1, 4, 3, 9, 9, 0, 2, 1, 6),
    ("real_freq_bits4", 1, 3, 2, 11, 10, 1, 1, 0, 4),
    ("real_bits12", 1, 4, 3, 10, 10, 0, 0, 0, 12),
    ("real_bits16_freq_mse", 1, 3, 2, 9, 11, 1, 2, 1, 16),
]


def real_valued():
    """tests/golden/qconv_real.npz: real-valued inputs / filters for every SFC variant."""
    arrays = {}
    rng = np.random.default_rng(0x5FC2)
    for tag, B, C, OC, H, W, asc, fsc, srch, bits in REAL_CASES:
        x = rng.normal(size=(B, C, H, W))
        arrays[f"{tag}/x"] = x
        arrays[f"{tag}/meta"] = np.array([asc, fsc, srch, bits], np.int64)
        for v in VARIANTS + LARGE_R:
            R = ob.spec(v, source="ref")["R"]
            w = rng.normal(size=(OC, C, R, R))
            pad = R // 2
            out, rep = ob.ref_quantized_fast_conv2d(x, w, v, pad, bits, asc, fsc, srch)
            arrays[f"{tag}/{v}/w"] = w
            arrays[f"{tag}/{v}/out"] = out
            arrays[f"{tag}/{v}/report"] = np.array([rep["mse"], rep["signal_energy"], rep["snr_db"],
                                                    rep["saturations"], rep["values_quantized"], pad], np.float64)
            arrays[f"{tag}/{v}/direct"] = ob.ref_direct_conv2d(x, w, pad)
            fo, mults = ob.ref_fast_conv2d(x, w, v, pad)  # the fp64 float path (conv.cpp:384-553)
            arrays[f"{tag}/{v}/fast"] = fo
            arrays[f"{tag}/{v}/fast_counts"] = mults
            fo, mults = ob.ref_fast_conv2d(x, w, v, pad, reduced=True)  # paired schedule (conv.cpp:466-509)
            arrays[f"{tag}/{v}/fast_red"] = fo
            arrays[f"{tag}/{v}/fast_red_counts"] = mults
    np.savez_compressed(os.path.join(HERE, "qconv_real.npz"), **arrays)
    print("wrote", len(arrays), "real-valued arrays")


# ------------------------------------------------------------------ command-line drop-in
# quantsim cases: CLI options (None = the CLI default) -> the reference's report per layer
CLI_QUANTSIM = [
    {"name": "defaults"},
    {"name": "sfc4_bits6_actfreq", "seed": "7", "algo": "sfc4-4x4-3x3", "bits": 6, "act": "frequency"},
    {"name": "sfc7_chfreq_mse_onef", "seed": "11", "algo": "sfc6-7x7-3x3", "fil": "channel-frequency",
     "search": "mse", "gen": "onef", "channels": 6, "out_channels": 5, "size": 30},
    {"name": "sfc5x5_freq_bits4", "seed": "0x2a", "algo": "sfc6-6x6-5x5", "bits": 4, "fil": "frequency",
     "padding": 2, "size": 19},
    {"name": "sfc7x7_onef", "seed": "99", "algo": "sfc6-4x4-7x7", "gen": "onef", "padding": 3, "size": 20},
    {"name": "bits2_saturating", "seed": "5", "bits": 2, "search": "mse", "channels": 3, "out_channels": 2},
    {"name": "layers_file", "seed": "1234", "bits": 7, "search": "mse", "layers": "cli_layers.json"},
    {"name": "env_seed", "env_seed": "12345", "act": "frequency", "fil": "channel-frequency"},
    {"name": "bits12", "seed": "21", "bits": 12},
    {"name": "bits16_onef_freq_mse", "seed": "22", "bits": 16, "gen": "onef", "act": "frequency",
     "fil": "channel-frequency", "search": "mse", "size": 16},
]
CLI_LAYERS = [  # tests/golden/cli_layers.json (the reference's layer-list format, tensor.cpp:66-90)
    {"name": "conv1", "in_channels": 3, "out_channels": 8, "height": 32, "width": 32, "kernel": 3, "padding": 1},
    {"name": "conv2", "in_channels": 8, "out_channels": 4, "height": 17, "width": 23, "kernel": 3},
    {"in_channels": 4, "out_channels": 4, "height": 12, "width": 12, "kernel": 3, "stride": 1, "padding": 1},
]
CLI_BENCH = [
    {"name": "defaults"},
    {"name": "reduced", "reduced": True},
    {"name": "sfc4_onef_reduced", "seed": "3", "algo": "sfc4-4x4-3x3", "gen": "onef", "size": 30,
     "channels": 5, "out_channels": 3, "reduced": True},
    {"name": "sfc5x5", "algo": "sfc6-6x6-5x5", "padding": 2, "size": 26, "channels": 4, "out_channels": 6},
]
CLI_DEFAULT_SEED = "0x5fc07751"  # sfconv_cli.cpp:30


def cli_quantsim_argv(c):
    """Command line of the drop-in CLI for a quantsim case (the environment goes separately)."""
    argv = (["--seed", c["seed"]] if "seed" in c else []) + ["quantsim"]
    for key, flag in [("algo", "--algo"), ("bits", "--bits"), ("act", "--act-scope"), ("fil", "--filter-scope"),
                      ("search", "--search"), ("gen", "--gen"), ("channels", "--channels"),
                      ("out_channels", "--out-channels"), ("size", "--size"), ("padding", "--padding")]:
        if key in c:
            argv += [flag, str(c[key])]
    if "layers" in c:
        argv += ["--layers", os.path.join("tests", "golden", c["layers"])]
    return argv


def cli_bench_argv(c):
    argv = (["--seed", c["seed"]] if "seed" in c else []) + ["bench"]
    for key, flag in [("algo", "--algo"), ("gen", "--gen"), ("channels", "--channels"),
                      ("out_channels", "--out-channels"), ("size", "--size"), ("padding", "--padding")]:
        if key in c:
            argv += [flag, str(c[key])]
    if c.get("reduced"):
        argv.append("--reduced")
    return argv


def cli_golden():
    """tests/golden/cli_golden.json: the reference library's quantsim reports / bench counters
    for the CLI cases, through oracle/_ref/cli_golden (inputs drawn as sfconv_cli.cpp does)."""
    import subprocess
    drv = os.path.join(ROOT, "oracle", "_ref", "cli_golden")
    if not os.path.exists(drv):
        raise SystemExit("oracle/_ref/cli_golden missing: run `make -C oracle` with /root/reference present")
    with open(os.path.join(HERE, "cli_layers.json"), "w") as f:
        json.dump(CLI_LAYERS, f, indent=2)
    out = {"quantsim": [], "bench": []}
    for c in CLI_QUANTSIM:
        algo = c.get("algo", "sfc6-6x6-3x3")
        R = ob.spec(algo, source="ref")["R"]
        if "layers" in c:
            specs = [f"{lc.get('name', f'layer{i}')}:{lc['in_channels']}:{lc['out_channels']}:{lc['height']}:"
                     f"{lc['width']}:{lc['kernel']}:{lc.get('padding', 0)}" for i, lc in enumerate(CLI_LAYERS)]
        else:
            size = c.get("size", 24)
            specs = [f"inline:{c.get('channels', 4)}:{c.get('out_channels', 4)}:{size}:{size}:{R}:{c.get('padding', 1)}"]
        seed = c.get("seed", c.get("env_seed", CLI_DEFAULT_SEED))
        res = subprocess.run([drv, "quantsim", seed, algo, str(c.get("bits", 8)), c.get("act", "tensor"),
                              c.get("fil", "channel"), c.get("search", "minmax"), c.get("gen", "gaussian"),
                              ",".join(specs)], check=True, capture_output=True, text=True).stdout
        rows = []
        for line in res.strip().splitlines():
            name, mse, snr, sat, vq = line.split()
            rows.append({"layer": name, "mse": float(mse), "snr_db": float(snr), "saturations": int(sat),
                         "values_quantized": int(vq)})
        env = {"SFC_SEED": c["env_seed"]} if "env_seed" in c else {}
        out["quantsim"].append({"name": c["name"], "argv": cli_quantsim_argv(c), "env": env, "seed": int(seed, 0),
                                "results": rows})
    for c in CLI_BENCH:
        algo = c.get("algo", "sfc6-6x6-3x3")
        seed = c.get("seed", CLI_DEFAULT_SEED)
        res = subprocess.run([drv, "bench", seed, algo, c.get("gen", "gaussian"), str(c.get("channels", 8)),
                              str(c.get("out_channels", 8)), str(c.get("size", 56)), str(c.get("padding", 1)),
                              "1" if c.get("reduced") else "0"], check=True, capture_output=True, text=True).stdout
        rel, mults, tiles = res.split()
        out["bench"].append({"name": c["name"], "argv": cli_bench_argv(c), "rel": float(rel),
                             "multiplications": int(mults), "tiles": int(tiles)})
    with open(os.path.join(HERE, "cli_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", len(out["quantsim"]), "quantsim and", len(out["bench"]), "bench cases")


def main():
    if "--cli" in sys.argv:
        return cli_golden()
    if "--large-r" in sys.argv:
        return large_r()
    if "--real" in sys.argv:
        return real_valued()
    if not ob.ref_available():
        raise SystemExit("oracle/_ref/libsfconv_ref.so missing: run `make -C oracle` with /root/reference present")
    js, h = ob.ref_catalog_json()
    full = json.loads(js)
    sel = [a for a in full["algorithms"] if a["name"] in VARIANTS]
    raw = {a["name"]: js[js.index('{"name":"' + a["name"]):] for a in sel}
    exact = {}
    for name, tail in raw.items():  # the exact substring of the reference export for each algorithm
        depth = 0
        for i, ch in enumerate(tail):
            depth += ch == "{"
            depth -= ch == "}"
            if depth == 0:
                exact[name] = tail[: i + 1]
                break
    with open(os.path.join(HERE, "catalog_3x3.json"), "w") as f:
        json.dump({"full_catalog_fnv1a64": f"{h:016x}", "algorithms": sel, "exact_text": exact}, f, indent=1)

    arrays = {}
    rng = np.random.default_rng(0x5FC0)
    for tag, B, C, OC, H, W, pad, lo, bits, asc, fsc, srch in CASES:
        x = rng.integers(lo, 128, size=(B, C, H, W), dtype=np.int8)
        w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
        arrays[f"{tag}/x"] = x
        arrays[f"{tag}/w"] = w
        arrays[f"{tag}/meta"] = np.array([pad, bits, asc, fsc, srch], np.int64)
        arrays[f"{tag}/direct"] = ob.ref_direct_conv2d(x, w, pad)
        for v in VARIANTS:
            out, rep = ob.ref_quantized_fast_conv2d(x, w, v, pad, bits, asc, fsc, srch)
            arrays[f"{tag}/{v}/out"] = out
            arrays[f"{tag}/{v}/report"] = np.array([rep["mse"], rep["signal_energy"], rep["snr_db"],
                                                    rep["saturations"], rep["values_quantized"]], np.float64)
            if tag == "small_p1":
                arrays[f"{tag}/{v}/u"] = ob.ref_transform_filters(w, v)
                xe = rng.integers(-128, 128, size=(1, 3, 14, 14), dtype=np.int8)
                arrays[f"{tag}/{v}/energy_x"] = xe
                arrays[f"{tag}/{v}/energy"] = ob.ref_frequency_energy(xe, v, 1)
    # scalar known answers (test_quant.cpp:34-72) evaluated by the reference
    kat_in = [(2.5, 1.0, 8), (3.5, 1.0, 8), (-2.5, 1.0, 8), (2.4999, 1.0, 8), (0.26, 0.1, 8), (127.4, 1.0, 8),
              (127.6, 1.0, 8), (-128.4, 1.0, 8), (-130.0, 1.0, 8), (9.0, 1.0, 4), (-9.0, 1.0, 4),
              (1020.0, 2040.0 / 127.0, 8), (-1020.0, 2040.0 / 127.0, 8)]
    arrays["kat/quantize_in"] = np.array(kat_in, np.float64)
    arrays["kat/quantize_out"] = np.array([ob.ref_quantize_value(*k) for k in kat_in], np.int64)
    grp = rng.normal(size=200)
    grp[0] = 12.0
    arrays["kat/scale_group"] = grp
    arrays["kat/scale_out"] = np.array([ob.ref_scale([-3.0, 1.0, 2.0], 8), ob.ref_scale([-3.0, 1.0, 2.0], 4),
                                        ob.ref_scale(np.zeros(10), 8), ob.ref_scale(grp, 8),
                                        ob.ref_scale(grp, 8, True), ob.ref_scale(grp, 4, True)], np.float64)
    np.savez_compressed(os.path.join(HERE, "qconv_cases.npz"), **arrays)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
