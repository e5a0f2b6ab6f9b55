"""The batch-sharded default path on the GPU: two processes (gloo, world size 2) share cuda:0
and drive the real CudaEngine -- absmax on the shard (V kept in the shard's workspace, or the
recompute schedule for multi-oc-block layers), all-reduce(MAX) of the int32 vmax, then
conv_kept / conv -- and the gathered output must equal a single forward of the whole batch
bit for bit (quant.cpp:171-172: the per-tensor scale is the whole batch's).

The exchange is host-mediated (gloo on a CPU copy of vmax), so neither rank's kernels wait
on the other's: the two processes only time-share the GPU.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


class _HostVmax:
    """CudaEngine with the exchanged vmax held on the host (gloo reduces CPU tensors)."""

    def __init__(self, eng):
        self.eng = eng

    def new_vmax(self, device):
        return torch.zeros(1, dtype=torch.int32)

    def absmax(self, x, vmax):
        d = vmax.to(x.device)
        self.eng.absmax(x, d)
        vmax.copy_(d.cpu())

    def conv(self, x, vmax, **outs):
        self.eng.conv(x, vmax.to(x.device), **outs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, x, w, variant, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_02913_b200 import sfconv as sc
        from paper_2407_02913_b200.distributed import CudaEngine, ShardedConv, shard_bounds
        dev = torch.device("cuda", 0)
        lo, hi = shard_bounds(x.shape[0], rank, world)
        xl = torch.from_numpy(x[lo:hi].copy()).to(dev)
        layer = sc.SfcLayer(variant, torch.from_numpy(w).to(dev))
        eng = CudaEngine(layer, 1)
        y = torch.empty((hi - lo, w.shape[0], x.shape[2], x.shape[3]), dtype=torch.int32, device=dev)
        vmax = ShardedConv(_HostVmax(eng)).forward(xl, y_int32=y)
        torch.cuda.synchronize()
        full = ShardedConv.gather_to_rank0(y.cpu(), x.shape[0])
        sched = layer.schedule(hi - lo, x.shape[2], x.shape[3], 1)
        if rank == 0:
            q.put((int(vmax.item()), full.numpy(), sched))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant,shape", [
    ("sfc6-6x6-3x3", (5, 64, 28, 28, 64)),     # one oc block: kept-V schedule (transform -> conv_kept)
    ("sfc4-4x4-3x3", (3, 32, 20, 20, 48)),
    ("sfc6-7x7-3x3", (4, 96, 14, 14, 320)),    # several oc blocks: recompute schedule (absmax -> conv)
])
def test_cuda_engine_sharded_equals_full_batch(cuda, variant, shape):
    from paper_2407_02913_b200 import sfconv as sc
    B, C, H, W, OC = shape
    rng = np.random.default_rng(B * 1000 + C)
    x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
    x[B - 1] //= 4                      # the last shard's local maximum is smaller than the global one
    w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
    layer = sc.SfcLayer(variant, torch.from_numpy(w).to(cuda))
    ws = layer.workspace(B, H, W, 1)
    y_full = torch.empty((B, OC, H, W), dtype=torch.int32, device=cuda)
    layer.forward(torch.from_numpy(x).to(cuda), ws, 1, y_int32=y_full)
    st = layer.stats(B, H, W, 1, ws)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, w, variant, q)) for r in range(2)]
    for p in procs:
        p.start()
    vmax, y, sched = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert vmax == st["vmax"]
    assert np.array_equal(y, y_full.cpu().numpy())
    assert sched["recompute"] == (OC > 256)
