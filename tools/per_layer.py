"""Per-layer device time of a workload's forward calls (CUDA events, L2 flushed before each
timed call) with direct-equivalent TOPS and the SURVEY §8(d) roofline time per layer.

    python tools/per_layer.py --workload 4 [--reps 5]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_02913_b200 import _lib, sfconv as sc, workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--workload", type=int, default=4)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
work = wl.WORKLOADS[a.workload]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
P_INT8, BW = 3.0e15, 6531.6e9
tot_ms = tot_roof = 0.0
print(f"{work.name}: layer  variant        shape                 ms      TOPS   roof_us  frac")
for i, L in enumerate(work.layers):
    x = torch.from_numpy(wl.activations(work.config, i, L)).cuda()
    w = torch.from_numpy(wl.weights(work.config, i, L)).cuda()
    ho = L.hw + 2 * L.pad - L.r + 1
    for v in work.variants:
        layer = sc.SfcLayer(v, w)
        ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
        outs = {}
        if work.requant:
            outs["out_i8"] = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int8, device="cuda")
        else:
            outs["y_int32"] = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int32, device="cuda")
        try:
            layer.forward(x, ws, L.pad, requant_scale=0.005, **outs)
        except _lib.SfcUnsupported:
            outs = {"y_int64": torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int64, device="cuda")}
            layer.forward(x, ws, L.pad, **outs)
        ms = 0.0
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            layer.forward(x, ws, L.pad, requant_scale=0.005, **outs)
            e1.record()
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1) / a.reps
        sp = layer.spec
        T, _, _ = wl.tile_grid(L, sp.M)
        ops = 2 * sp.K * sp.K * T * L.cin * L.cout
        ob = sum(t.numel() * t.element_size() for t in outs.values())
        byts = L.batch * L.cin * L.hw * L.hw + sp.K * sp.K * L.cin * L.cout + ob
        roof = max(ops / P_INT8, byts / BW) * 1e6
        tops = wl.direct_equivalent_ops(L) / (ms / 1e3) / 1e12
        tot_ms += ms
        tot_roof += roof
        print(f"  {i:2d} {v:14s} b{L.batch} {L.cin:3d}->{L.cout:3d} @{L.hw:3d}  {ms:8.3f} {tops:8.1f} {roof:8.1f} {roof / 1e3 / ms:5.2f}")
print(f"total {tot_ms:.3f} ms, step roofline fraction {tot_roof / 1e3 / tot_ms:.3f}")
