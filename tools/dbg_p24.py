"""Debug: decoded 24-bit pacc (layouts 2 / 1) vs int32 pacc on one small case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2407_02913_b200 import sfconv as sc
rng = np.random.default_rng(3)
B, C, OC, H, W = 1, 8, 8, 14, 14
x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
for variant in ("sfc4-4x4-3x3", "sfc6-6x6-3x3"):
    res = {}
    for name, env in (("u", {}), ("rows", {"SFC_OUT_MMA": "0"}), ("p32", {"SFC_P24": "0"})):
        for k in ("SFC_P24", "SFC_OUT_MMA"):
            os.environ.pop(k, None)
        os.environ.update(env)
        layer = sc.SfcLayer(variant, torch.from_numpy(w).cuda())
        xt = torch.from_numpy(x).cuda()
        ws = layer.workspace(B, H, W, 1)
        y = torch.empty((B, OC, H, W), dtype=torch.int32, device="cuda")
        layer.forward(xt, ws, 1, y_int32=y)
        torch.cuda.synchronize()
        _, p = layer.views(B, H, W, 1, ws)
        res[name] = (y.cpu().numpy(), p.cpu().numpy(), layer.schedule(B, H, W, 1))
        print(variant, name, res[name][2])
    for name in ("u", "rows"):
        yd = (res[name][0] != res["p32"][0]).sum()
        pd = res[name][1] != res["p32"][1]
        print(variant, name, "y mismatches", yd, "pacc mismatches", pd.sum(), "of", pd.size)
        if pd.sum():
            idx = np.argwhere(pd)[:12]
            for f, t, oc in idx:
                a, b = int(res[name][1][f, t, oc]), int(res["p32"][1][f, t, oc])
                print("   f t oc", f, t, oc, "got", a, hex(a & 0xffffff), "want", b, hex(b & 0xffffff))
            fs = np.unique(np.argwhere(pd)[:, 0]); ts = np.unique(np.argwhere(pd)[:, 1]); ocs = np.unique(np.argwhere(pd)[:, 2])
            print("   f:", fs[:20], "t:", ts[:20], "oc:", ocs[:20])
