"""Profiling driver: W warm-up + 1 profiled forward of one workload/variant (default
config 2, sfc6-6x6-3x3).  Use with ncu -k regex:... -s <skip> -c <count>."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_02913_b200 import sfconv as sc, workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--workload", type=int, default=2)
ap.add_argument("--layer", type=int, default=0)
ap.add_argument("--variant", default="sfc6-6x6-3x3")
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--i8", action="store_true", help="int8 requant output only (configs 3/4)")
a = ap.parse_args()
work = wl.WORKLOADS[a.workload]
L = work.layers[a.layer]
x = torch.from_numpy(wl.activations(a.workload, a.layer, L)).cuda()
w = torch.from_numpy(wl.weights(a.workload, a.layer, L)).cuda()
layer = sc.SfcLayer(a.variant, w)
ho = L.hw + 2 * L.pad - L.r + 1
ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
out = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.float32, device="cuda")
kw = dict(y_int32=torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int32, device="cuda"), out_f32=out)
if a.i8:
    kw = dict(out_i8=torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int8, device="cuda"), requant_scale=0.004)
try:
    layer.forward(x, ws, L.pad, **kw)
except sc.SfcUnsupported if hasattr(sc, "SfcUnsupported") else Exception:
    kw = dict(y_int64=torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int64, device="cuda"), out_f32=out)
for _ in range(a.iters):
    layer.forward(x, ws, L.pad, **kw)
torch.cuda.synchronize()
print("ok")
