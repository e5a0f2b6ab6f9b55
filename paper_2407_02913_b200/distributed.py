"""Batch-sharded multi-GPU execution of one quantized SFC layer (one process per GPU).

SURVEY.md §8(e): tiles and images are independent, so the batch is split across ranks
with no data-path collective.  The single exchange needed for bit-exactness is the
per-tensor activation scale, which the reference takes over the *whole* batch
(proj/src/quant.cpp:171-172): every rank runs the absmax pre-pass on its shard, then one
all-reduce(MAX) of an int32 (order-free, exact) makes the scale global before
quantization.  Outputs are gathered to rank 0 only for checking, outside timing.

The engine is injected so the same host logic runs on the GPU (``CudaEngine`` over the
C-ABI, NCCL) and in the CPU multi-process tests (gloo + a test engine).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def shard_bounds(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced batch shard [lo, hi) of `rank` (sizes differ by at most one)."""
    base, rem = divmod(batch, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def _global_rank(group, rank: int) -> int:
    return rank if group is None else dist.get_global_rank(group, rank)


class CudaEngine:
    """Adapter of sfconv.SfcLayer to the engine protocol used by ShardedConv."""

    def __init__(self, layer, pad: int):
        self.layer, self.pad = layer, pad
        self._ws = {}

    def new_vmax(self, device):
        return torch.zeros(1, dtype=torch.int32, device=device)

    def _workspace(self, x):
        key = tuple(x.shape)
        if key not in self._ws:
            n, _, h, w = x.shape
            self._ws[key] = self.layer.workspace(n, h, w, self.pad)
        return self._ws[key]

    def _recompute(self, x) -> bool:
        """The single-GPU forward's schedule for this shard (sfc_conv_schedule): recompute V
        from x after the exchange, or keep it from the absmax pass."""
        n, _, h, w = x.shape
        return self.layer.schedule(n, h, w, self.pad)["recompute"]

    def absmax(self, x, vmax):
        """Local absmax; V is kept in the shard's workspace for conv() unless the schedule
        recomputes it."""
        if self._recompute(x):
            self.layer.absmax(x, vmax, self.pad)
        else:
            self.layer.transform(x, vmax, self._workspace(x), self.pad)

    def conv(self, x, vmax, **outs):
        if self._recompute(x):
            self.layer.conv(x, vmax, self._workspace(x), self.pad, **outs)
        else:
            self.layer.conv_kept(tuple(x.shape), vmax, self._workspace(x), self.pad, **outs)

    # -- general QuantConfig (per-frequency scopes, MseGrid): see ShardedConv.forward_general
    @property
    def mse(self) -> bool:
        return self.layer.search == 1

    def general_prepare(self, x):
        return self.layer.general_prepare(x, self._workspace(x), self.pad)

    def general_count(self) -> int:
        """Number of activation maxima exchanged: K*K for PerFrequency, else 1."""
        return self.layer.spec.K ** 2 if self.layer.act_scope == 1 else 1

    def general_mse(self, x, err_in):
        n, _, h, w = x.shape
        groups = self.layer.spec.K ** 2 if self.layer.act_scope == 1 else 1
        err_out = torch.empty((groups, 101), dtype=torch.float64, device=x.device)
        self.layer.general_mse_partial(n, h, w, self.pad, self._workspace(x), err_in, err_out)
        return err_out

    def general_conv(self, x, err, **outs):
        n, _, h, w = x.shape
        self.layer.general_conv(n, h, w, self.pad, self._workspace(x), err, **outs)


@dataclass
class ShardedConv:
    engine: object
    group: object = None

    def forward(self, x_local, **outs):
        """absmax on the local shard -> all-reduce(MAX) -> quantize/contract/transform locally.
        A rank whose shard is empty (batch < world) contributes a zero maximum and still joins
        the exchange, so no rank waits on a collective another one never reaches."""
        vmax = self.engine.new_vmax(x_local.device)
        empty = x_local.shape[0] == 0
        if not empty:
            self.engine.absmax(x_local, vmax)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(vmax, op=dist.ReduceOp.MAX, group=self.group)
        if not empty:
            self.engine.conv(x_local, vmax, **outs)
        return vmax

    def forward_general(self, x_local, **outs):
        """A non-default QuantConfig (PerFrequency scopes, MseGrid; quant.cpp:163-229): the
        activation scales are functions of the whole batch.  Local maxima -> all-reduce(MAX)
        (fp64 bit patterns, exact); for MseGrid each candidate's error is ONE sequential fp64
        sum over the batch in tile order (quant.cpp:19-30), so the sums travel rank to rank in
        batch order (each rank continues the previous rank's accumulators over its shard) and
        the last rank's complete sums are broadcast; every rank then picks the same scales and
        quantizes / contracts / transforms its shard.  Bitwise the full-batch result."""
        empty = x_local.shape[0] == 0  # batch < world: join every exchange with a neutral part
        if empty:
            maxima = torch.zeros(self.engine.general_count(), dtype=torch.int64, device=x_local.device)
        else:
            maxima = self.engine.general_prepare(x_local)
        multi = dist.is_initialized() and dist.get_world_size(self.group) > 1
        if multi:
            dist.all_reduce(maxima, op=dist.ReduceOp.MAX, group=self.group)
        elif empty:
            raise ValueError("empty batch")
        err = None
        if self.engine.mse:
            err_in = None
            if multi:
                world, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
                if rank > 0:
                    err_in = torch.empty((maxima.numel(), 101), dtype=torch.float64, device=x_local.device)
                    dist.recv(err_in, src=_global_rank(self.group, rank - 1), group=self.group)
                # an empty shard adds no terms: the running sums pass through unchanged
                err = err_in if empty else self.engine.general_mse(x_local, err_in)
                if rank < world - 1:
                    dist.send(err, dst=_global_rank(self.group, rank + 1), group=self.group)
                dist.broadcast(err, src=_global_rank(self.group, world - 1), group=self.group)
            else:
                err = self.engine.general_mse(x_local, None)
        if not empty:
            self.engine.general_conv(x_local, err, **outs)
        return maxima

    @staticmethod
    def gather_to_rank0(t_local, batch: int, group=None):
        """Concatenate every rank's output shard on rank 0 (checking only; not timed)."""
        if not dist.is_initialized() or dist.get_world_size(group) == 1:
            return t_local
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        shapes = [shard_bounds(batch, r, world) for r in range(world)]
        bufs = [t_local.new_empty((hi - lo,) + tuple(t_local.shape[1:])) for lo, hi in shapes]
        if t_local.device.type == "cpu":  # gloo has no gather of unequal sizes; use all_gather of padded
            maxn = max(hi - lo for lo, hi in shapes)
            pad = t_local.new_zeros((maxn,) + tuple(t_local.shape[1:]))
            pad[: t_local.shape[0]] = t_local
            allp = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(allp, pad, group=group)
            bufs = [p[: hi - lo] for p, (lo, hi) in zip(allp, shapes)]
        else:
            dist.all_gather(bufs, t_local.contiguous(), group=group)
        return torch.cat(bufs, 0) if rank == 0 else None
