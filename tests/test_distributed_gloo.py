"""World-size-2 gloo test of the batch-sharded host logic (paper_2407_02913_b200.distributed).

Each rank holds half of the batch; the per-tensor activation scale must still be the
full-batch one (quant.cpp:171-172), obtained by all-reduce(MAX) of the local absmax.  The
engine here is the CPU oracle (test infrastructure) standing in for the CUDA engine, so the
exchange/sharding/gather logic is exercised exactly as on the GPU path.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_02913_b200.distributed import ShardedConv, shard_bounds


class OracleEngine:
    def __init__(self, w, spec, pad):
        self.w, self.spec, self.pad = w, spec, pad

    def new_vmax(self, device):
        return torch.zeros(1, dtype=torch.int32, device=device)

    def absmax(self, x, vmax):
        from oracle import bindings as ob
        r = ob.quantized_conv(x.numpy(), self.w, self.spec, self.pad, want=(), threads=1)
        vmax.copy_(torch.maximum(vmax, torch.tensor([r["report"]["vmax"]], dtype=torch.int32)))

    def conv(self, x, vmax, y_int32=None):
        from oracle import bindings as ob
        r = ob.quantized_conv(x.numpy(), self.w, self.spec, self.pad, want=("y_int",), threads=1,
                              vmax_override=int(vmax.item()))
        y_int32.copy_(torch.from_numpy(r["y_int"].astype(np.int32)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, x, w, spec, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_bounds(x.shape[0], rank, world)
        xl = torch.from_numpy(x[lo:hi].copy())
        y = torch.empty((hi - lo, w.shape[0], x.shape[2], x.shape[3]), dtype=torch.int32)
        sc = ShardedConv(OracleEngine(w, spec, 1))
        vmax = sc.forward(xl, y_int32=y)
        full = ShardedConv.gather_to_rank0(y, x.shape[0])
        if rank == 0:
            q.put((int(vmax.item()), full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("spec", ["sfc6-6x6-3x3", "sfc4-4x4-3x3"])
def test_sharded_equals_full_batch(spec):
    from oracle import bindings as ob
    rng = np.random.default_rng(11)
    x = rng.integers(-128, 128, size=(3, 4, 13, 13), dtype=np.int8)   # odd batch: ragged shards
    x[2] *= 0                                                        # rank 1's shard has a smaller local max
    x[2, 0, 5, 5] = 3
    w = rng.integers(-127, 128, size=(5, 4, 3, 3), dtype=np.int8)
    full = ob.quantized_conv(x, w, spec, 1, want=("y_int",))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, w, spec, q)) for r in range(2)]
    for p in procs:
        p.start()
    vmax, y = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert vmax == full["report"]["vmax"]
    assert np.array_equal(y.astype(np.int64), full["y_int"])


def test_shard_bounds_cover_batch():
    for batch in range(1, 20):
        for world in range(1, 9):
            b = [shard_bounds(batch, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == batch
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1
