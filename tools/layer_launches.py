"""One warm forward per layer of a workload (configs 3/4: int8 requant outputs, else int32 y),
each bracketed by NVTX-free markers so an ncu launch list can be split per layer.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file out.csv python tools/layer_launches.py --workload 4
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_02913_b200 import sfconv as sc, workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--workload", type=int, default=4)
ap.add_argument("--variant", default=None)
a = ap.parse_args()
work = wl.WORKLOADS[a.workload]
for i, L in enumerate(work.layers):
    x = torch.from_numpy(wl.activations(a.workload, i, L)).cuda()
    w = torch.from_numpy(wl.weights(a.workload, i, L)).cuda()
    ho = L.hw + 2 * L.pad - L.r + 1
    for v in ([a.variant] if a.variant else work.variants):
        layer = sc.SfcLayer(v, w)
        ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
        if work.requant:
            kw = dict(out_i8=torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int8, device="cuda"),
                      requant_scale=0.004)
        else:
            kw = dict(y_int32=torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int32, device="cuda"))
        layer.forward(x, ws, L.pad, **kw)
        torch.cuda.synchronize()
        print(f"layer {i} {v} {L.cin}->{L.cout}@{L.hw} sched={layer.schedule(L.batch, L.hw, L.hw, L.pad)}",
              flush=True)
        del ws, layer
        torch.cuda.empty_cache()
