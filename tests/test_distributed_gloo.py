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


# ------------------------------------------------------------------ general QuantConfig
class NumpyGeneralEngine:
    """The shard steps of ShardedConv.forward_general restated on the host (test
    infrastructure): V = B^T x B exactly (quant.cpp:44-93), the activation maxima as fp64 bit
    patterns, MseGrid sums as one sequential Python-float fold per candidate in the
    reference's value order (quant.cpp:19-30, 168-181), and the shard's output from the C
    oracle quantizing with the exchanged full-batch scales."""

    def __init__(self, w, spec, pad, bits, asc, fsc, srch):
        from oracle import bindings as ob
        self.w, self.spec, self.pad, self.bits = w, spec, pad, bits
        self.asc, self.fsc, self.srch = asc, fsc, srch
        self.sp = ob.spec(spec)
        self.mse = srch == 1
        self.scales = None

    def _v(self, x):  # [T, C, F] int64, tiles in (b, ti, tj) order
        sp = self.sp
        K, n, M, R = sp["K"], sp["n"], sp["M"], sp["R"]
        bt = sp["BT"].astype(np.int64)
        B, C, H, W = x.shape
        HO, WO = H + 2 * self.pad - R + 1, W + 2 * self.pad - R + 1
        th, tw = -(-HO // M), -(-WO // M)
        xp = np.zeros((B, C, th * M + n, tw * M + n), np.int64)
        xp[:, :, self.pad:self.pad + H, self.pad:self.pad + W] = x
        out = []
        for b in range(B):
            for ti in range(th):
                for tj in range(tw):
                    win = xp[b, :, ti * M:ti * M + n, tj * M:tj * M + n]
                    out.append(np.einsum("kr,crs,ls->ckl", bt, win, bt).reshape(C, K * K))
        return np.stack(out)

    def _qmax(self):
        return float((1 << (self.bits - 1)) - 1)

    def general_prepare(self, x):
        self.v = self._v(x.numpy())
        a = np.abs(self.v).astype(np.float64)
        m = a.max(axis=(0, 1)) if self.asc == 1 else np.array([a.max()])
        return torch.from_numpy(m.astype(np.float64).view(np.int64).copy())

    def _base(self, maxima, g):
        return max(float(np.int64(maxima[g]).view(np.float64)) / self._qmax(), 1e-8)

    def general_mse(self, x, err_in):
        import math
        qmax, qmin = self._qmax(), -self._qmax() - 1.0
        groups = self.v.shape[2] if self.asc == 1 else 1
        err = np.zeros((groups, 101)) if err_in is None else err_in.numpy().copy()
        for g in range(groups):
            base = self._base(self._maxima, g)
            vals = self.v[:, :, g].ravel() if self.asc == 1 else self.v.ravel()
            for cand in range(101):
                s = base if cand == 0 else max(base * (0.3 + (0.7 * (cand - 1)) / 99.0), 1e-8)
                e = err[g, cand]
                for v in vals.tolist():
                    q = min(qmax, max(qmin, float(np.rint(v / s))))
                    d = v - q * s
                    e = e + d * d
                err[g, cand] = e
        return torch.from_numpy(err)

    def general_conv(self, x, err, out_f64=None):
        from oracle import bindings as ob
        groups = self._maxima.numel()
        scales = []
        for g in range(groups):
            base = self._base(self._maxima, g)
            best = base
            if err is not None:
                e = err.numpy()
                best_err = e[g, 0]
                for cand in range(1, 101):
                    if e[g, cand] < best_err:
                        best_err, best = e[g, cand], max(base * (0.3 + (0.7 * (cand - 1)) / 99.0), 1e-8)
            scales.append(best)
        self.scales = np.array(scales)
        r = ob.quantized_conv(x.numpy(), self.w, self.spec, self.pad, self.bits, self.asc, self.fsc, self.srch,
                              want=("out",), threads=1, act_scale_override=self.scales)
        out_f64.copy_(torch.from_numpy(r["out"]))


class _MaximaHook:
    """Lets the numpy engine see the all-reduced maxima (the CUDA engine reads them from its
    workspace, where the all-reduce writes in place)."""

    def __init__(self, eng):
        self.eng = eng
        self.mse = eng.mse

    def general_prepare(self, x):
        self.eng._maxima = self.eng.general_prepare(x)
        return self.eng._maxima

    def general_mse(self, x, err_in):
        return self.eng.general_mse(x, err_in)

    def general_conv(self, x, err, **outs):
        return self.eng.general_conv(x, err, **outs)

    def general_count(self):
        return self.eng.sp["K"] ** 2 if self.eng.asc == 1 else 1


def _general_worker(rank, world, port, x, w, spec, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_bounds(x.shape[0], rank, world)
        xl = torch.from_numpy(x[lo:hi].copy())
        eng = NumpyGeneralEngine(w, spec, 1, *cfg)
        out = torch.empty((hi - lo, w.shape[0], x.shape[2], x.shape[3]), dtype=torch.float64)
        ShardedConv(_MaximaHook(eng)).forward_general(xl, out_f64=out)
        full = ShardedConv.gather_to_rank0(out, x.shape[0])
        if rank == 0:
            q.put((eng.scales, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [(8, 1, 0, 0), (6, 0, 2, 1), (8, 1, 1, 1), (12, 0, 0, 1)],
                         ids=["actfreq", "chfreq_mse", "actfreq_freq_mse", "bits12_mse"])
def test_sharded_general_quantconfig_equals_full_batch(cfg):
    """The general QuantConfig over world_size 2 (gloo): per-frequency maxima all-reduced, the
    MseGrid sums chained rank 0 -> rank 1 and broadcast; the scales and the gathered output equal
    the full-batch oracle's bit for bit (odd batch: ragged shards; the shards differ in range)."""
    from oracle import bindings as ob
    bits, asc, fsc, srch = cfg
    rng = np.random.default_rng(21 + sum(cfg))
    x = rng.integers(-128, 128, size=(3, 2, 7, 7), dtype=np.int8)
    x[2] //= 8                                                      # rank 1's shard has smaller values
    w = rng.integers(-127, 128, size=(3, 2, 3, 3), dtype=np.int8)
    spec = "sfc4-4x4-3x3"
    full = ob.quantized_conv(x, w, spec, 1, bits, asc, fsc, srch, want=("out",))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_general_worker, args=(r, 2, port, x, w, spec, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    scales, out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert np.array_equal(scales, full["act_scale"])
    assert np.array_equal(out, full["out"])


def _empty_worker(rank, world, port, x, w, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_bounds(x.shape[0], rank, world)
        xl = torch.from_numpy(x[lo:hi].copy())
        y = torch.empty((hi - lo, w.shape[0], x.shape[2], x.shape[3]), dtype=torch.int32)
        vmax = ShardedConv(OracleEngine(w, "sfc6-6x6-3x3", 1)).forward(xl, y_int32=y)
        full = ShardedConv.gather_to_rank0(y, x.shape[0])
        eng = NumpyGeneralEngine(w, "sfc4-4x4-3x3", 1, 8, 1, 0, 1)
        out = torch.empty((hi - lo, w.shape[0], x.shape[2], x.shape[3]), dtype=torch.float64)
        ShardedConv(_MaximaHook(eng)).forward_general(xl, out_f64=out)
        gen = ShardedConv.gather_to_rank0(out, x.shape[0])
        if rank == 0:
            q.put((int(vmax.item()), full.numpy(), eng.scales, gen.numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_batch_smaller_than_world():
    """batch 2 over 3 ranks: rank 2's shard is empty.  It joins the all-reduce with a zero
    maximum (and passes the MseGrid sums through), so no rank blocks, and the gathered
    results equal the full-batch oracle's (empty shards used to raise before the
    collective and hang the other ranks)."""
    from oracle import bindings as ob
    rng = np.random.default_rng(5)
    x = rng.integers(-128, 128, size=(2, 3, 7, 7), dtype=np.int8)
    w = rng.integers(-127, 128, size=(2, 3, 3, 3), dtype=np.int8)
    full = ob.quantized_conv(x, w, "sfc6-6x6-3x3", 1, want=("y_int",))
    gen = ob.quantized_conv(x, w, "sfc4-4x4-3x3", 1, 8, 1, 0, 1, want=("out",))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_empty_worker, args=(r, 3, port, x, w, q)) for r in range(3)]
    for p in procs:
        p.start()
    vmax, y, scales, out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert vmax == full["report"]["vmax"]
    assert np.array_equal(y.astype(np.int64), full["y_int"])
    assert np.array_equal(scales, gen["act_scale"])
    assert np.array_equal(out, gen["out"])
