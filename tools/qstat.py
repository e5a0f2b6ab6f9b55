import sys; sys.path.insert(0, ".")
import torch
from paper_2407_02913_b200 import sfconv as sc, workloads as wl
for w in (2, 3, 4, 5):
    work = wl.WORKLOADS[w]
    for li in ((0,) if w != 3 and w != 4 else range(len(work.layers))):
        L = work.layers[li]
        if L.batch * L.cin * L.hw * L.hw > 2e9: continue
        x = torch.from_numpy(wl.activations(w, li, L)).cuda(); wt = torch.from_numpy(wl.weights(w, li, L)).cuda()
        for v in work.variants:
            layer = sc.SfcLayer(v, wt); ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
            ho = L.hw + 2 * L.pad - L.r + 1
            y = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int64, device="cuda")
            layer.forward(x, ws, L.pad, y_int64=y); torch.cuda.synchronize()
            st = layer.stats(L.batch, L.hw, L.hw, L.pad, ws)
            print(work.name, li, v, "vmax", st["vmax"], "exact", st["fast_quantizer_exact"], flush=True)
