"""Fraction of plane-2 rows the GEMM flags (sparse plane 2 of unit-major P) per layer of a workload.

    python tools/p2_flags.py --workload 4 [--batch 16]
"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2407_02913_b200 import sfconv as sc, workloads as wl
from paper_2407_02913_b200._lib import check, lib

ap = argparse.ArgumentParser()
ap.add_argument("--workload", type=int, default=4)
ap.add_argument("--batch", type=int, default=16)
a = ap.parse_args()
work = wl.WORKLOADS[a.workload]
for i, L in enumerate(work.layers):
    b = min(L.batch, a.batch)
    x = torch.from_numpy(wl.activations(work.config, i, L, batch=b)).cuda()
    w = torch.from_numpy(wl.weights(work.config, i, L)).cuda()
    ho = L.hw + 2 * L.pad - L.r + 1
    for v in work.variants:
        layer = sc.SfcLayer(v, w)
        if layer.schedule(b, L.hw, L.hw, L.pad)["p_layout"] != 2:
            print(i, v, "layout", layer.schedule(b, L.hw, L.hw, L.pad)["p_layout"])
            continue
        ws = layer.workspace(b, L.hw, L.hw, L.pad)
        y = torch.empty((b, L.cout, ho, ho), dtype=torch.int32, device="cuda")
        layer.forward(x, ws, L.pad, y_int32=y)
        torch.cuda.synchronize()
        vq, pa = ctypes.c_void_p(), ctypes.c_void_p()
        geom = np.zeros(6, np.int64)
        check(lib().sfc_conv_views(layer._h, b, L.hw, L.hw, L.pad, sc._ptr(ws), ws.numel(), ctypes.byref(vq), ctypes.byref(pa),
                                   geom.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        T, Tpad, Cpad, OCpad = (int(t) for t in geom[:4])
        F = layer.spec.K ** 2
        n_ob, n_tg = OCpad // 32, Tpad // 4
        fl = sc._wrap_device(pa.value + 3 * F * Tpad * OCpad, (n_ob, n_tg // 8, F, 8), torch.uint8, x.device)
        fl = (fl.permute(0, 1, 3, 2).reshape(-1, F)[: , :] != 0).float()
        per_f = fl.mean(0).cpu().numpy()
        _, p = layer.views(b, L.hw, L.hw, L.pad, ws)
        pmax = p.abs().amax(dim=(1, 2)).cpu().numpy()
        print(f"layer {i} {v} b{b} {L.cin}->{L.cout}@{L.hw}: flagged rows {per_f.mean():.4f}; f with >1% flagged: "
              f"{[(int(f), round(float(per_f[f]), 3)) for f in np.argsort(-per_f)[:12] if per_f[f] > 0.01]}; max|P| DC {pmax[0]}, "
              f"median over f {np.median(pmax):.0f}")
