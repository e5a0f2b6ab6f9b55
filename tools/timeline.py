"""Device timeline of one forward (timeline build): per kernel, first CTA entry, first CTA
past its dependency wait and last CTA exit, relative to the first kernel's entry (us).

    make -C paper_2407_02913_b200/csrc TIMELINE=1
    python tools/timeline.py --workload 2        (loads paper_2407_02913_b200/libsfc_b200_tl.so)
"""
import argparse, ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SFC_B200_LIB", os.path.join(ROOT, "paper_2407_02913_b200", "libsfc_b200_tl.so"))
import torch
from paper_2407_02913_b200 import _lib, sfconv as sc, workloads as wl

NAMES = ["reset", "absmax", "quantize", "gemm", "output", "-"]
ap = argparse.ArgumentParser()
ap.add_argument("--workload", type=int, default=2)
ap.add_argument("--layer", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
L = wl.WORKLOADS[a.workload].layers[a.layer]
x = torch.from_numpy(wl.activations(a.workload, a.layer, L)).cuda()
w = torch.from_numpy(wl.weights(a.workload, a.layer, L)).cuda()
lib = _lib.lib()
buf = (ctypes.c_uint64 * 24)()
ho = L.hw + 2 * L.pad - L.r + 1
NONE = 2**64 - 1
for v in wl.WORKLOADS[a.workload].variants:
    layer = sc.SfcLayer(v, w)
    ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
    out = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.float32, device="cuda")
    kw = dict(y_int32=torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int32, device="cuda"), out_f32=out)
    try:
        layer.forward(x, ws, L.pad, **kw)
    except _lib.SfcUnsupported:
        kw = dict(y_int64=torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int64, device="cuda"), out_f32=out)
    for _ in range(5):
        layer.forward(x, ws, L.pad, **kw)
    for r in range(a.reps):
        assert lib.sfc_debug_timeline(buf, 1) == 0
        torch.cuda._sleep(200_000)  # ~100 us: every launch below is queued before the device reaches it
        layer.forward(x, ws, L.pad, **kw)
        assert lib.sfc_debug_timeline(buf, 1) == 0
        t = [(buf[3 * k], buf[3 * k + 1], buf[3 * k + 2]) for k in range(6)]
        t0 = t[0][2]  # the reset kernel's exit (its entry includes the spin of the sleep kernel)
        rel = lambda z: (z - t0) / 1e3 if z != NONE else float("nan")
        row = "  ".join(f"{NAMES[k]} {rel(s):5.1f}/{rel(wt):5.1f}/{rel(e):5.1f}" for k, (s, wt, e) in enumerate(t)
                        if s != NONE)
        print(f"{v} [{wl.WORKLOADS[a.workload].name}] entry/waited/exit us: {row}   end {rel(max(e for _, _, e in t)):.1f}")
