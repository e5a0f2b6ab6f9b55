"""Host time per forward vs device time, eager vs CUDA-graph replay (config 2, sfc6-6x6-3x3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_02913_b200 import sfconv as sc, workloads as wl
L = wl.WORKLOADS[2].layers[0]
x = torch.from_numpy(wl.activations(2, 0, L)).cuda()
w = torch.from_numpy(wl.weights(2, 0, L)).cuda()
layer = sc.SfcLayer("sfc6-6x6-3x3", w)
ws = layer.workspace(8, 28, 28, 1)
y = torch.empty((8, 128, 28, 28), dtype=torch.int32, device="cuda")
out = torch.empty((8, 128, 28, 28), dtype=torch.float32, device="cuda")
for _ in range(10):
    layer.forward(x, ws, 1, y_int32=y, out_f32=out)
torch.cuda.synchronize()
n = 200
t = time.perf_counter()
for _ in range(n):
    layer.forward(x, ws, 1, y_int32=y, out_f32=out)
host = (time.perf_counter() - t) / n
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    layer.forward(x, ws, 1, y_int32=y, out_f32=out)
e1.record(); torch.cuda.synchronize()
print(f"eager: host {host*1e6:.1f} us/call, device {e0.elapsed_time(e1)/n*1e3:.1f} us/call")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    layer.forward(x, ws, 1, y_int32=y, out_f32=out)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        layer.forward(x, ws, 1, y_int32=y, out_f32=out)
torch.cuda.synchronize()
y_ref = y.clone()
for _ in range(10):
    g.replay()
torch.cuda.synchronize()
assert torch.equal(y, y_ref)
e0.record()
for _ in range(n):
    g.replay()
e1.record(); torch.cuda.synchronize()
print(f"graph: device {e0.elapsed_time(e1)/n*1e3:.1f} us/call")
