"""Per-stage device time per tile vs batch: does a stage speed up when its intermediate
(kept V / vq / P) fits in L2?  Stages run back to back (no flush between them), L2 flushed
before each call.  SFC_FORWARD_RECOMPUTE etc. select schedules as usual.

    python tools/l2_probe.py --shape 512,512,14 --batches 8,16,32,64,128,256
"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2407_02913_b200 import sfconv as sc
from paper_2407_02913_b200._lib import lib

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="512,512,14")
ap.add_argument("--batches", default="8,16,32,64,128,256")
ap.add_argument("--variant", default="sfc6-6x6-3x3")
ap.add_argument("--i8", action="store_true")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
cin, cout, hw = (int(v) for v in a.shape.split(","))
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.integers(-127, 128, size=(cout, cin, 3, 3), dtype=np.int8)).cuda()
layer = sc.SfcLayer(a.variant, w)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
L_ = lib()
for B in (int(b) for b in a.batches.split(",")):
    x = torch.from_numpy(rng.integers(-128, 128, size=(B, cin, hw, hw), dtype=np.int8)).cuda()
    ws = layer.workspace(B, hw, hw, 1)
    if a.i8:
        outs = {"out_i8": torch.empty((B, cout, hw, hw), dtype=torch.int8, device="cuda")}
    else:
        outs = {"y_int32": torch.empty((B, cout, hw, hw), dtype=torch.int32, device="cuda")}
    sched = layer.schedule(B, hw, hw, 1)
    rec = sched["recompute"]
    vmax = torch.zeros(1, dtype=torch.int32, device="cuda")
    masks = ((1, "reset"), (2, "quant"), (4, "gemm"), (8, "out")) if rec else ((1, "reset"), (4 | 16, "gemm"), (8 | 16, "out"))
    acc = {}
    for r in range(a.reps + 1):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(len(masks) + 2)]
        o = sc.Outputs(*(sc._ptr(outs.get(k)) for k in ("y_int32", "y_int64", "out_f32", "out_f64", "out_i8")), 0.004)
        vmax.zero_()
        e[0].record(st)
        if rec:
            layer.absmax(x, vmax, 1)
        else:
            layer.transform(x, vmax, ws, 1)
        e[1].record(st)
        for si, (mask, _) in enumerate(masks):
            sc.check(L_.sfc_conv_int8_stages(layer._h, sc._ptr(x), B, hw, hw, 1, sc._ptr(vmax), sc._ptr(ws), ws.numel(),
                                             ctypes.byref(o), mask, ctypes.c_void_p(st.cuda_stream)))
            e[2 + si].record(st)
        e[-1].synchronize()
        if r == 0:
            continue
        acc["absmax"] = acc.get("absmax", 0) + e[0].elapsed_time(e[1]) / a.reps
        for si, (_, nme) in enumerate(masks):
            acc[nme] = acc.get(nme, 0) + e[1 + si].elapsed_time(e[2 + si]) / a.reps
    T = layer.stats(B, hw, hw, 1, ws)["tiles"]
    pmb = T * cout * layer.spec.K ** 2 * 3 / 1e6
    print(f"B={B:4d} T={T:6d} P={pmb:7.1f}MB sched={sched} " +
          " ".join(f"{k}={v * 1e3:8.1f}us({v * 1e6 / T:6.2f}ns/t)" for k, v in acc.items()), flush=True)
    del ws, x, outs
    torch.cuda.empty_cache()
