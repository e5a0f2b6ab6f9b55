"""Per-stage device time of the two forward paths (kept V vs recompute), one layer.

    python tools/stage_paths.py --workload 5 [--variant sfc6-6x6-3x3] [--layer 0]

Each stage is launched alone between CUDA events (no PDL overlap), averaged over reps,
L2 flushed before every rep.  Prints one line per stage plus the chained forwards.
"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_02913_b200 import _lib, sfconv as sc, workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--workload", type=int, default=5)
ap.add_argument("--variant", default=None)
ap.add_argument("--layer", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
work = wl.WORKLOADS[a.workload]
L = work.layers[a.layer]
variants = [a.variant] if a.variant else list(work.variants)
x = torch.from_numpy(wl.activations(a.workload, a.layer, L)).cuda()
w = torch.from_numpy(wl.weights(a.workload, a.layer, L)).cuda()
ho = L.hw + 2 * L.pad - L.r + 1
lib = _lib.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def timeit(fn, reps=a.reps):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1e3


for v in variants:
    layer = sc.SfcLayer(v, w)
    ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
    y = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int32, device="cuda")
    vmax = torch.zeros(1, dtype=torch.int32, device="cuda")
    o = _lib.Outputs(ctypes.c_void_p(y.data_ptr()), None, None, None, None, 0.0)

    def stages(mask):
        _lib.check(lib.sfc_conv_int8_stages(layer._h, ctypes.c_void_p(x.data_ptr()), L.batch, L.hw, L.hw, L.pad,
                                            ctypes.c_void_p(vmax.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                            ws.numel(), ctypes.byref(o), mask,
                                            ctypes.c_void_p(st.cuda_stream)))

    res = {}
    res["forward(default)"] = timeit(lambda: layer.forward(x, ws, L.pad, y_int32=y))
    res["absmax(no keep)"] = timeit(lambda: (vmax.zero_(), layer.absmax(x, vmax, L.pad)))
    res["act quant(recompute)"] = timeit(lambda: stages(2))
    res["gemm(vq TMA)"] = timeit(lambda: stages(4))
    res["output"] = timeit(lambda: stages(8))
    res["recompute chain"] = timeit(lambda: (vmax.zero_(), layer.absmax(x, vmax, L.pad), layer.conv(
        x, vmax, ws, L.pad, y_int32=y)))
    res["absmax(keep V)"] = timeit(lambda: (vmax.zero_(), layer.transform(x, vmax, ws, L.pad)))
    res["gemm(kept V fused)"] = timeit(lambda: stages(4 | 16))
    print(f"{work.name} layer {a.layer} {v}: " + "  ".join(f"{k} {t:.1f}" for k, t in res.items()), flush=True)
