"""Repeat one forward many times and report run-to-run differences of y (race hunting).

    python tools/stress_repeat.py --workload 5 --variant sfc6-7x7-3x3 --reps 20
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2407_02913_b200 import _lib, sfconv as sc, workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--workload", type=int, default=5)
ap.add_argument("--layer", type=int, default=0)
ap.add_argument("--variant", default="sfc6-7x7-3x3")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--fresh", action="store_true", help="new layer + workspace each repetition")
a = ap.parse_args()
L = wl.WORKLOADS[a.workload].layers[a.layer]
x = torch.from_numpy(wl.activations(a.workload, a.layer, L)).cuda()
w = torch.from_numpy(wl.weights(a.workload, a.layer, L)).cuda()
ho = L.hw + 2 * L.pad - L.r + 1
ref = None
bad = 0
for r in range(a.reps):
    if r == 0 or a.fresh:
        layer = sc.SfcLayer(a.variant, w)
        ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
    y = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int64, device="cuda")
    try:
        layer.forward(x, ws, L.pad, y_int64=y)
    except _lib.SfcUnsupported:
        raise
    torch.cuda.synchronize()
    yc = y.cpu().numpy()
    if ref is None:
        ref = yc
        continue
    d = np.argwhere(yc != ref)
    if len(d):
        bad += 1
        print(f"rep {r}: {len(d)} mismatches; b {np.unique(d[:, 0])[:8]} oc {np.unique(d[:, 1])[:16]} "
              f"h {np.unique(d[:, 2])} w {np.unique(d[:, 3])}")
print(f"{a.variant} workload {a.workload}: {bad} of {a.reps - 1} repetitions differ from the first")
