"""Race hunt: forward once, then re-run individual stages on the finished workspace and
compare y / P across repetitions.

    python tools/stress_stages.py --workload 5 --variant sfc6-7x7-3x3
"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2407_02913_b200 import _lib, sfconv as sc, workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--workload", type=int, default=5)
ap.add_argument("--variant", default="sfc6-7x7-3x3")
ap.add_argument("--reps", type=int, default=8)
a = ap.parse_args()
L = wl.WORKLOADS[a.workload].layers[0]
x = torch.from_numpy(wl.activations(a.workload, 0, L)).cuda()
w = torch.from_numpy(wl.weights(a.workload, 0, L)).cuda()
ho = L.hw + 2 * L.pad - L.r + 1
layer = sc.SfcLayer(a.variant, w)
ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
y = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int64, device="cuda")
layer.forward(x, ws, L.pad, y_int64=y)
torch.cuda.synchronize()
vq0, p0 = [t.clone() for t in layer.views(L.batch, L.hw, L.hw, L.pad, ws)]
y0 = y.clone()
vmax = torch.tensor([layer.stats(L.batch, L.hw, L.hw, L.pad, ws)["vmax"]], dtype=torch.int32, device="cuda")
lib = _lib.lib()


def stages(mask):
    o = _lib.Outputs(None, ctypes.c_void_p(y.data_ptr()), None, None, None, 0.0)
    _lib.check(lib.sfc_conv_int8_stages(layer._h, ctypes.c_void_p(x.data_ptr()), L.batch, L.hw, L.hw, L.pad,
                                        ctypes.c_void_p(vmax.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                        ctypes.byref(o), mask, None))
    torch.cuda.synchronize()


for name, mask in (("output only", 8), ("gemm only", 4), ("gemm+output", 12), ("act only", 2)):
    diffs = []
    for r in range(a.reps):
        y.zero_()
        stages(mask)
        vq, p = layer.views(L.batch, L.hw, L.hw, L.pad, ws)
        diffs.append((int((y != y0).sum()) if mask & 8 else -1, int((p != p0).sum()), int((vq != vq0).sum())))
    print(f"{name:12s} (y, P, vq) mismatches vs first forward: {diffs}")
