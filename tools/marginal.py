"""Marginal steady-state cost of each kernel of a PDL-chained forward (config 2, one variant)."""
import os, subprocess, sys
code = r'''
import os, sys, torch
sys.path.insert(0, ".")
from paper_2407_02913_b200 import sfconv as sc, workloads as wl
v = sys.argv[1]
L = wl.WORKLOADS[2].layers[0]
x = torch.from_numpy(wl.activations(2, 0, L)).cuda(); w = torch.from_numpy(wl.weights(2, 0, L)).cuda()
layer = sc.SfcLayer(v, w); ws = layer.workspace(8, 28, 28, 1)
ho = 28
y = torch.empty((8,128,ho,ho), dtype=torch.int32, device="cuda"); out = torch.empty((8,128,ho,ho), dtype=torch.float32, device="cuda")
for _ in range(20): layer.forward(x, ws, 1, y_int32=y, out_f32=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.Stream(); G = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(G, stream=s):
        for _ in range(50): layer.forward(x, ws, 1, y_int32=y, out_f32=out)
torch.cuda.synchronize()
for _ in range(3): G.replay()
torch.cuda.synchronize()
n = 10; e0.record()
for _ in range(n): G.replay()
e1.record(); torch.cuda.synchronize(); print(e0.elapsed_time(e1) / n / 50 * 1e3)
'''
for v in ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3"]:
    res = {}
    for name, mask in (("absmax", 0), ("+act", 2), ("+gemm", 6), ("+output", 14)):
        env = dict(os.environ, SFC_DEBUG_FORWARD_MASK=str(mask))
        r = subprocess.run([sys.executable, "-c", code, v], env=env, capture_output=True, text=True)
        res[name] = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
    print(v, {k: (round(x, 1) if isinstance(x, float) else x) for k, x in res.items()})
