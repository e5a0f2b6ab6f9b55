"""Python mirror of the reference's quantized-SFC interface on the B200 device path.

Names, argument meaning and error behaviour follow proj/include/sfconv/{spec,conv,quant}.hpp
so parity tests read like the reference's own (proj/tests/test_quant.cpp).  Tensors are
torch tensors; activations and weights must hold int8 integer values (the values the
reference receives as doubles).  Everything numerical runs in libsfc_b200.so on the GPU;
the scalar helpers quantize_value / scale_minmax / scale_mse_grid are host utilities
with the reference's exact double semantics (quant.cpp:102-134).
"""
from __future__ import annotations

import ctypes
import enum
import math
import os
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from ._lib import Outputs, check, lib


class ActScaleScope(enum.IntEnum):
    PerTensor = 0
    PerFrequency = 1


class FilterScaleScope(enum.IntEnum):
    PerChannel = 0
    PerFrequency = 1
    PerChannelFrequency = 2


class ScaleSearch(enum.IntEnum):
    MinMax = 0
    MseGrid = 1


@dataclass
class QuantConfig:
    """quant.hpp:20-25."""
    bits: int = 8
    act_scope: ActScaleScope = ActScaleScope.PerTensor
    filter_scope: FilterScaleScope = FilterScaleScope.PerChannel
    search: ScaleSearch = ScaleSearch.MinMax


@dataclass
class QuantReport:
    """quant.hpp:27-34, plus the exact integer accumulator and the scales."""
    output: torch.Tensor                 # float32 [B, OC, HO, WO] (device)
    mse: float = 0.0
    signal_energy: float = 0.0
    snr_db: float = 0.0
    saturations: int = 0
    values_quantized: int = 0
    y_int: torch.Tensor | None = None    # int32 [B, OC, HO, WO] = sum_kl A A pacc
    act_scale: float = 0.0
    filter_scales: np.ndarray | None = None


@dataclass
class CorrectionTerm:
    out: int
    desired: int
    wrapped: int
    tap: int


@dataclass
class AlgorithmSpec:
    """spec.hpp:36-62 (integer matrices as numpy int64)."""
    name: str
    N: int
    M: int
    R: int
    offset: int
    K: int
    n_in: int
    a_denom: int
    BT: np.ndarray
    G: np.ndarray
    A: np.ndarray
    corrections: list = field(default_factory=list)
    _mults_full: int = 0
    _mults_reduced: int = 0
    _handle: int = 0

    def mults_full(self) -> int:
        return self._mults_full

    def mults_reduced(self) -> int:
        return self._mults_reduced

    def complexity_pct(self) -> float:
        return 100.0 * self._mults_reduced / (self.M * self.M * self.R * self.R)


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


# ----------------------------------------------------------------------------------- catalog
@lru_cache(maxsize=None)
def catalog_algorithm(name: str) -> AlgorithmSpec:
    """catalog.cpp:275-287: derive, exactness-gate and cache; unknown names raise ValueError."""
    h = ctypes.c_void_p()
    check(lib().sfc_plan_create(name.encode(), ctypes.byref(h)))
    dims = np.zeros(10, np.int64)
    check(lib().sfc_plan_dims(h, dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    K, n, M, R, N, off, den, nc, mf, mr = (int(v) for v in dims)
    bt = np.zeros((K, n), np.int64)
    g = np.zeros((K, R), np.int64)
    a = np.zeros((K, M), np.int64)
    p = ctypes.POINTER(ctypes.c_int64)
    check(lib().sfc_plan_matrices(h, bt.ctypes.data_as(p), g.ctypes.data_as(p), a.ctypes.data_as(p)))
    corr = []
    for k in range(K - nc, K):
        d = int(np.nonzero(bt[k] == 1)[0][0])
        wr = int(np.nonzero(bt[k] == -1)[0][0])
        corr.append(CorrectionTerm(int(np.nonzero(a[k])[0][0]), d, wr, int(np.nonzero(g[k])[0][0])))
    return AlgorithmSpec(name, N, M, R, off, K, n, den, bt, g, a, corr, mf, mr, h.value)


def catalog_names():
    """The SFC entries of the reference catalog, in its order (catalog.cpp:246-250)."""
    return ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3", "sfc6-6x6-5x5", "sfc6-4x4-7x7"]


def catalog_export_json() -> tuple[str, int]:
    buf = ctypes.create_string_buffer(1 << 18)
    h = ctypes.c_uint64()
    check(lib().sfc_catalog_json(buf, len(buf), ctypes.byref(h)))
    return buf.value.decode(), h.value


# ----------------------------------------------------------------------------------- scalars
def quantize_value(v: float, scale: float, bits: int, saturated: list | None = None) -> int:
    """quant.cpp:102-115: RNE (np.rint == nearbyint) then clamp to the signed b-bit range."""
    qmax, qmin = (1 << (bits - 1)) - 1, -(1 << (bits - 1))
    q = int(np.rint(np.float64(v) / np.float64(scale)))
    if q > qmax or q < qmin:
        q = qmax if q > qmax else qmin
        if saturated is not None:
            saturated[0] += 1
    return q


def scale_minmax(values, bits: int) -> float:
    """quant.cpp:117-120."""
    v = np.asarray(values, np.float64)
    m = float(np.max(np.abs(v))) if v.size else 0.0
    return max(m / float((1 << (bits - 1)) - 1), 1e-8)


def _group_mse(v: np.ndarray, scale: float, bits: int) -> float:
    qmax, qmin = float((1 << (bits - 1)) - 1), -float(1 << (bits - 1))
    err = 0.0
    for x in v:  # sequential, like quant.cpp:19-30
        q = min(qmax, max(qmin, float(np.rint(x / scale))))
        d = x - q * scale
        err += d * d
    return err


def scale_mse_grid(values, bits: int) -> float:
    """quant.cpp:122-134."""
    v = np.asarray(values, np.float64).ravel()
    base = scale_minmax(v, bits)
    best, best_err = base, _group_mse(v, base, bits)
    for i in range(100):
        s = max(base * (0.3 + 0.7 * float(i) / 99.0), 1e-8)
        e = _group_mse(v, s, bits)
        if e < best_err:
            best, best_err = s, e
    return best


# ----------------------------------------------------------------------------------- device
def is_int8_valued(t) -> bool:
    """True if every value of t is an integer in [-128, 127] (the int8 fast path applies)."""
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.asarray(t))
    if t.dtype == torch.int8:
        return True
    td = t.to(torch.float64)
    return bool(torch.all(td == torch.round(td))) and not bool((td < -128).any()) and not bool((td > 127).any())


def as_f64_device(t, device=None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.asarray(t))
    dev = device or (t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    return t.to(dev, torch.float64).contiguous()


def as_int8_device(t, what: str, device=None) -> torch.Tensor:
    """Accept int8 tensors as-is; accept other dtypes only if every value is an int8 integer."""
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.asarray(t))
    dev = device or (t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    if t.dtype == torch.int8:
        return t.to(dev).contiguous()
    td = t.to(dev, torch.float64)
    if not bool(torch.all(td == torch.round(td))) or bool((td < -128).any()) or bool((td > 127).any()):
        raise ValueError(f"{what}: the B200 path needs int8-valued tensors (integers in [-128, 127])")
    return td.to(torch.int8).contiguous()


class SfcLayer:
    """One conv layer on the device: offline-transformed, quantized filters (sfc_layer_t)."""

    def __init__(self, spec: AlgorithmSpec | str, filters: torch.Tensor, bits: int = 8,
                 filter_scope: int = FilterScaleScope.PerChannel, search: int = ScaleSearch.MinMax, stream=None,
                 act_scope: int = ActScaleScope.PerTensor, real: bool = False):
        """real=True: fp64 filters of any value (sfc_layer_create_f64, the reference's own
        arithmetic order); the layer then runs the fp64 epilogue (no y_int)."""
        self.spec = catalog_algorithm(spec) if isinstance(spec, str) else spec
        if filters.dim() != 4 or filters.shape[2] != self.spec.R or filters.shape[3] != self.spec.R:
            raise ValueError("filter shape does not match algorithm")
        w = as_f64_device(filters) if real else as_int8_device(filters, "filters")
        self.device = w.device
        self.OC, self.IC = int(w.shape[0]), int(w.shape[1])
        self.bits = bits
        self.act_scope, self.filter_scope, self.search = int(act_scope), int(filter_scope), int(search)
        # anything but {PerTensor, PerChannel, MinMax} at <= 8 bits is the fp64 parity path (no
        # y_int); 9-16 bits contract integer-valued fp64 operands exactly (fp64 GEMM)
        self.general = real or bits > 8 or (self.act_scope, self.filter_scope, self.search) != (0, 0, 0)
        self.real = real
        h = ctypes.c_void_p()
        create = lib().sfc_layer_create_f64 if real else lib().sfc_layer_create_ex
        with torch.cuda.device(self.device):
            check(create(ctypes.c_void_p(self.spec._handle), _ptr(w), self.OC, self.IC, bits, self.act_scope,
                         self.filter_scope, self.search, ctypes.c_void_p(_stream_ptr(stream)), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and _lib._lib is not None:
                _lib._lib.sfc_layer_destroy(h)
        except Exception:  # interpreter shutdown: module globals may already be gone
            pass
        self._h = None

    # -- filter side
    def filter_scales(self):
        sf = np.zeros(self.OC, np.float64)
        um = np.zeros(self.OC, np.int32)
        check(lib().sfc_layer_filter_scales(self._h, sf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            um.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        return sf, um

    def filter_scales_native(self) -> np.ndarray:
        """Filter scales as the scope defines them (OC, K*K or OC*K*K; quant.cpp:193-219)."""
        n = ctypes.c_int64()
        check(lib().sfc_layer_filter_scales_native(self._h, None, ctypes.byref(n)))
        out = np.zeros(n.value, np.float64)
        check(lib().sfc_layer_filter_scales_native(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                                   ctypes.byref(n)))
        return out

    def act_scales(self, n, h, w, pad, ws, stream=None) -> np.ndarray:
        """Activation scales of the last call (1 or K*K)."""
        cnt = ctypes.c_int64()
        check(lib().sfc_conv_act_scales(self._h, n, h, w, pad, _ptr(ws), ws.numel(), None, ctypes.byref(cnt),
                                        ctypes.c_void_p(_stream_ptr(stream))))
        out = np.zeros(cnt.value, np.float64)
        check(lib().sfc_conv_act_scales(self._h, n, h, w, pad, _ptr(ws), ws.numel(), out.ctypes.data_as(
            ctypes.POINTER(ctypes.c_double)), ctypes.byref(cnt), ctypes.c_void_p(_stream_ptr(stream))))
        return out

    def filter_saturations(self) -> int:
        c = ctypes.c_int64()
        check(lib().sfc_layer_saturations(self._h, ctypes.byref(c)))
        return c.value

    def uq(self) -> torch.Tensor:
        """Quantized transformed filters as int8 [F, OC, IC] (a copy of the device buffer)."""
        p, icp, ocp = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        check(lib().sfc_layer_uq(self._h, ctypes.byref(p), ctypes.byref(icp), ctypes.byref(ocp)))
        F = self.spec.K ** 2
        full = _wrap_device(p.value, (F, ocp.value, icp.value), torch.int8, self.device)
        return full[:, : self.OC, : self.IC].clone()

    # -- per call
    def workspace_size(self, n, h, w, pad) -> int:
        b = ctypes.c_size_t()
        check(lib().sfc_conv_workspace_size(self._h, n, h, w, pad, ctypes.byref(b)))
        return b.value

    def workspace(self, n, h, w, pad) -> torch.Tensor:
        return torch.empty(self.workspace_size(n, h, w, pad), dtype=torch.uint8, device=self.device)

    def absmax(self, x: torch.Tensor, vmax: torch.Tensor, pad: int, stream=None):
        n, c, h, w = x.shape
        if c != self.IC:
            raise ValueError("input channel count does not match filters")
        check(lib().sfc_act_absmax(self._h, _ptr(x), n, h, w, pad, _ptr(vmax), ctypes.c_void_p(_stream_ptr(stream))))

    def transform(self, x: torch.Tensor, vmax: torch.Tensor, ws: torch.Tensor, pad: int, stream=None):
        """absmax pre-pass that keeps V in `ws` for conv_kept (sfc_act_transform)."""
        n, c, h, w = x.shape
        if c != self.IC:
            raise ValueError("input channel count does not match filters")
        check(lib().sfc_act_transform(self._h, _ptr(x), n, h, w, pad, _ptr(vmax), _ptr(ws), ws.numel(),
                                      ctypes.c_void_p(_stream_ptr(stream))))

    def conv_kept(self, shape, vmax: torch.Tensor, ws: torch.Tensor, pad: int, y_int32=None, y_int64=None,
                  out_f32=None, out_i8=None, requant_scale: float = 0.0, stream=None, out_f64=None):
        """Quantize the V kept by transform() with the (all-reduced) vmax, contract, output transform."""
        n, c, h, w = shape
        o = Outputs(_ptr(y_int32), _ptr(y_int64), _ptr(out_f32), _ptr(out_f64), _ptr(out_i8), float(requant_scale))
        check(lib().sfc_conv_kept(self._h, n, h, w, pad, _ptr(vmax), _ptr(ws), ws.numel(), ctypes.byref(o),
                                  ctypes.c_void_p(_stream_ptr(stream))))

    def conv(self, x: torch.Tensor, vmax: torch.Tensor, ws: torch.Tensor, pad: int, y_int32=None, y_int64=None,
             out_f32=None, out_i8=None, requant_scale: float = 0.0, stream=None, out_f64=None):
        n, c, h, w = x.shape
        if c != self.IC:
            raise ValueError("input channel count does not match filters")
        o = Outputs(_ptr(y_int32), _ptr(y_int64), _ptr(out_f32), _ptr(out_f64), _ptr(out_i8), float(requant_scale))
        check(lib().sfc_conv_int8(self._h, _ptr(x), n, h, w, pad, _ptr(vmax), _ptr(ws), ws.numel(), ctypes.byref(o),
                                  ctypes.c_void_p(_stream_ptr(stream))))

    def forward(self, x: torch.Tensor, ws: torch.Tensor, pad: int, y_int32=None, y_int64=None, out_f32=None,
                out_i8=None, requant_scale: float = 0.0, stream=None, out_f64=None):
        n, c, h, w = x.shape
        if c != self.IC:
            raise ValueError("input channel count does not match filters")
        o = Outputs(_ptr(y_int32), _ptr(y_int64), _ptr(out_f32), _ptr(out_f64), _ptr(out_i8), float(requant_scale))
        check(lib().sfc_conv_forward(self._h, _ptr(x), n, h, w, pad, _ptr(ws), ws.numel(), ctypes.byref(o),
                                     ctypes.c_void_p(_stream_ptr(stream))))

    def forward_f64(self, x: torch.Tensor, ws: torch.Tensor, pad: int, out_f32=None, out_f64=None, out_i8=None,
                    requant_scale: float = 0.0, stream=None):
        """Real-valued fp64 input x (sfc_conv_forward_f64)."""
        n, c, h, w = x.shape
        if c != self.IC:
            raise ValueError("input channel count does not match filters")
        x = as_f64_device(x, self.device)
        o = Outputs(None, None, _ptr(out_f32), _ptr(out_f64), _ptr(out_i8), float(requant_scale))
        check(lib().sfc_conv_forward_f64(self._h, _ptr(x), n, h, w, pad, _ptr(ws), ws.numel(), ctypes.byref(o),
                                         ctypes.c_void_p(_stream_ptr(stream))))

    # -- the general QuantConfig on a batch shard (sfc_general_*: see include/sfc_b200.h)
    def general_prepare(self, x: torch.Tensor, ws: torch.Tensor, pad: int, stream=None) -> torch.Tensor:
        """absmax keeps V; returns this shard's activation maxima (int64 view of the fp64 bit
        patterns in the workspace: an all-reduce(MAX) over ranks is the exact global max)."""
        n, c, h, w = x.shape
        if c != self.IC:
            raise ValueError("input channel count does not match filters")
        ptr, cnt = ctypes.c_void_p(), ctypes.c_int()
        check(lib().sfc_general_prepare(self._h, _ptr(x), n, h, w, pad, _ptr(ws), ws.numel(), ctypes.byref(ptr),
                                        ctypes.byref(cnt), ctypes.c_void_p(_stream_ptr(stream))))
        return _wrap_device(ptr.value, (cnt.value,), torch.int64, self.device)

    def general_mse_partial(self, n, h, w, pad, ws, err_in, err_out, stream=None):
        """MseGrid sums [groups, 101] (fp64) continued over this shard from err_in (None: batch start)."""
        check(lib().sfc_general_mse_partial(self._h, n, h, w, pad, _ptr(ws), ws.numel(), _ptr(err_in), _ptr(err_out),
                                            ctypes.c_void_p(_stream_ptr(stream))))

    def general_conv(self, n, h, w, pad, ws, err=None, out_f32=None, out_f64=None, out_i8=None,
                     requant_scale: float = 0.0, stream=None):
        o = Outputs(None, None, _ptr(out_f32), _ptr(out_f64), _ptr(out_i8), float(requant_scale))
        check(lib().sfc_general_conv(self._h, n, h, w, pad, _ptr(ws), ws.numel(), _ptr(err), ctypes.byref(o),
                                     ctypes.c_void_p(_stream_ptr(stream))))

    def stats(self, n, h, w, pad, ws, stream=None) -> dict:
        s = np.zeros(6, np.int64)
        check(lib().sfc_conv_stats(self._h, n, h, w, pad, _ptr(ws), ws.numel(), s.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                   ctypes.c_void_p(_stream_ptr(stream))))
        return dict(act_scale=float(s[0:1].view(np.float64)[0]), vmax=int(s[1]), saturations=int(s[2]),
                    fast_quantizer_exact=bool(s[3]), values_quantized=int(s[4]), tiles=int(s[5]))

    def schedule(self, n, h, w, pad) -> dict:
        """The schedule forward() picks (sfc_conv_schedule): recompute (bool), p_layout (int)."""
        r, pl = ctypes.c_int(), ctypes.c_int()
        check(lib().sfc_conv_schedule(self._h, n, h, w, pad, ctypes.byref(r), ctypes.byref(pl)))
        return {"recompute": bool(r.value), "p_layout": pl.value}

    def views(self, n, h, w, pad, ws):
        """(vq int8 [F, T, IC], pacc int32 [F, T, OC]) views of the workspace after conv();
        pacc is None when the layer's P is chunked (never materialised whole)."""
        vq, pa = ctypes.c_void_p(), ctypes.c_void_p()
        geom = np.zeros(6, np.int64)
        check(lib().sfc_conv_views(self._h, n, h, w, pad, _ptr(ws), ws.numel(), ctypes.byref(vq), ctypes.byref(pa),
                                   geom.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        T, Tpad, Cpad, OCpad = (int(v) for v in geom[:4])
        F = self.spec.K ** 2
        blocked = ctypes.c_int()
        check(lib().sfc_conv_schedule(self._h, n, h, w, pad, None, ctypes.byref(blocked)))
        if blocked.value == 3:  # Cin <= 4: vq compact [F][T][4], P never materialised
            return _wrap_device(vq.value, (F, T, 4), torch.int8, self.device)[:, :, : self.IC], None
        vqt = _wrap_device(vq.value, (F, Tpad, Cpad), torch.int8, self.device)[:, :T, : self.IC]
        if not pa.value:
            return vqt, None
        if blocked.value == 2:  # unit-major 24-bit P (sfc_kernels.hpp pu_offset), pre-swizzled (a copy)
            n_ob, n_tg = OCpad // 32, Tpad // 4
            raw = _wrap_device(pa.value, (n_ob, 3, F, n_tg, 128), torch.uint8, self.device)
            f = torch.arange(F, device=self.device)[:, None, None]
            lb = torch.arange(128, device=self.device)[None, None, :]
            src = ((((lb >> 4) ^ (f & 7)) << 4) | (lb & 15)).expand(n_ob, 3, F, n_tg, 128)
            lg = torch.gather(raw, 4, src).to(torch.int32)  # [ob][plane][f][tg][tt * 32 + oc]
            hi = (((lg[:, 2] & 0xFF) ^ 0x80) - 0x80) * 65536
            p = (lg[:, 0] & 0xFF) | ((lg[:, 1] & 0xFF) << 8)
            if os.environ.get("SFC_P2_DENSE", "0")[:1] == "1":
                p = p | hi
            else:  # sparse plane 2: P + 2^15 stored; rows of plane 2 exist where the flag byte is set
                fl = _wrap_device(pa.value + 3 * F * Tpad * OCpad, (n_ob, n_tg // 8, F, 8), torch.uint8, self.device)
                fl = fl.permute(0, 2, 1, 3).reshape(n_ob, F, n_tg, 1) != 0
                p = p + torch.where(fl, hi, torch.zeros_like(hi)) - 32768
            p = p.view(n_ob, F, n_tg, 4, 32).permute(1, 2, 3, 0, 4).reshape(F, n_tg * 4, n_ob * 32)
            return vqt, p[:, :T, : self.OC]
        if blocked.value == 1:  # 24-bit rows of three byte planes b0 | b1 | b2 (a copy)
            raw = _wrap_device(pa.value, (F, Tpad, 3 * OCpad), torch.uint8, self.device)
            b0 = raw[:, :, :OCpad].to(torch.int32) & 0xFF  # (the wrapped view may be signed bytes)
            b1 = raw[:, :, OCpad:2 * OCpad].to(torch.int32) & 0xFF
            b2 = raw[:, :, 2 * OCpad:].contiguous().view(torch.int8).to(torch.int32)
            return vqt, (b0 | (b1 << 8) | (b2 << 16))[:, :T, : self.OC]
        pat = _wrap_device(pa.value, (F, Tpad, OCpad), torch.int32, self.device)[:, :T, : self.OC]
        return vqt, pat


def _wrap_device(ptr: int, shape, dtype, device) -> torch.Tensor:
    """Zero-copy torch view of device memory owned by the library / workspace."""
    itemsize = torch.empty((), dtype=dtype).element_size()
    n = int(np.prod(shape))

    class _Arr:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": {1: "|i1", 4: "<i4", 8: "<i8"}[itemsize], "data": (ptr, False), "version": 3,
            "strides": None,
        }

    with torch.cuda.device(device):
        return torch.as_tensor(_Arr(), device=device).view(*shape)


def direct_conv2d(input, filters, stride: int = 1, padding: int = 0) -> torch.Tensor:
    """conv.cpp:320-350 for int8-valued tensors; exact (int32 accumulation), returned as float64."""
    x = as_int8_device(input, "input")
    w = as_int8_device(filters, "filters", x.device)
    if x.dim() != 4 or w.dim() != 4:
        raise ValueError("conv2d expects 4-d NCHW tensors")
    if w.shape[2] != w.shape[3]:
        raise ValueError("conv2d expects square filters")
    if x.shape[1] != w.shape[1]:
        raise ValueError("input channel count does not match filters")
    if stride < 1:
        raise ValueError("stride must be positive")
    B, C, H, W = x.shape
    OC, _, R, _ = w.shape
    HO, WO = (H + 2 * padding - R) // stride + 1, (W + 2 * padding - R) // stride + 1
    if HO <= 0 or WO <= 0 or H + 2 * padding < R or W + 2 * padding < R:
        raise ValueError("filter larger than padded input")
    out = torch.empty((B, OC, HO, WO), dtype=torch.int32, device=x.device)
    check(lib().sfc_direct_conv_int8(_ptr(x), B, C, H, W, _ptr(w), OC, R, stride, padding, _ptr(out),
                                     ctypes.c_void_p(_stream_ptr())))
    return out.to(torch.float64)


def transform_filters(filters, spec: AlgorithmSpec) -> torch.Tensor:
    """conv.cpp:352-382: G f G^T per (oc, ic) -> float64 [OC, IC, K, K] (exact integers)."""
    if filters.dim() != 4 or filters.shape[2] != spec.R or filters.shape[3] != spec.R:
        raise ValueError("filter shape does not match algorithm")
    w = as_int8_device(filters, "filters")
    OC, IC = int(w.shape[0]), int(w.shape[1])
    u = torch.empty((OC, IC, spec.K, spec.K), dtype=torch.int32, device=w.device)
    check(lib().sfc_transform_filters_int8(ctypes.c_void_p(spec._handle), _ptr(w), OC, IC, _ptr(u),
                                           ctypes.c_void_p(_stream_ptr())))
    return u.to(torch.float64)


def frequency_energy(input, spec: AlgorithmSpec, padding: int = 0) -> np.ndarray:
    """quant.cpp:136-150: mean V^2 per frequency over every tile and channel."""
    x = as_int8_device(input, "input")
    B, C, H, W = x.shape
    HO, WO = H + 2 * padding - spec.R + 1, W + 2 * padding - spec.R + 1
    if HO <= 0 or WO <= 0:
        raise ValueError("filter larger than padded input")
    s = torch.zeros(spec.K * spec.K, dtype=torch.int64, device=x.device)
    check(lib().sfc_frequency_energy_int8(ctypes.c_void_p(spec._handle), _ptr(x), B, C, H, W, padding, _ptr(s),
                                          ctypes.c_void_p(_stream_ptr())))
    groups = B * (-(-HO // spec.M)) * (-(-WO // spec.M)) * C
    return s.cpu().numpy().astype(np.float64) / float(groups)


def _snr_db(sig: float, err: float) -> float:
    """10 log10(sig / max(err, 1e-300)) with C++ semantics (log10(0) = -inf; quant.cpp:291)."""
    r = sig / max(err, 1e-300)
    return 10.0 * math.log10(r) if r > 0 else float("-inf")


def quantized_fast_conv2d(input, filters, spec: AlgorithmSpec, padding: int, config: QuantConfig = QuantConfig(),
                          report: bool = True) -> QuantReport:
    """quant.cpp:152-293 on the device.  Raises ValueError for bits outside [2, 16] (quant.cpp:155-156)."""
    if config.bits < 2 or config.bits > 16:
        raise ValueError("quantization width must be between 2 and 16 bits")
    if not (is_int8_valued(input) and is_int8_valued(filters)):
        return _quantized_fast_conv2d_real(input, filters, spec, padding, config, report)
    x = as_int8_device(input, "input")
    if x.dim() != 4 or filters.dim() != 4:
        raise ValueError("conv2d expects 4-d NCHW tensors")
    if filters.shape[1] != x.shape[1]:
        raise ValueError("input channel count does not match filters")
    B, C, H, W = x.shape
    if H + 2 * padding - spec.R + 1 <= 0 or W + 2 * padding - spec.R + 1 <= 0:
        raise ValueError("filter larger than padded input")
    layer = SfcLayer(spec, filters, config.bits, config.filter_scope, config.search,
                     act_scope=config.act_scope)
    HO, WO = H + 2 * padding - spec.R + 1, W + 2 * padding - spec.R + 1
    ws = layer.workspace(B, H, W, padding)
    out = torch.empty((B, layer.OC, HO, WO), dtype=torch.float32, device=x.device)
    y = None
    if layer.general:  # per-frequency dequantisation in fp64: no integer y (quant.cpp:258-263)
        layer.forward(x, ws, padding, out_f32=out)
    else:
        y = torch.empty((B, layer.OC, HO, WO), dtype=torch.int32, device=x.device)
        try:
            layer.forward(x, ws, padding, y_int32=y, out_f32=out)
        except _lib.SfcUnsupported:  # the int32 bound does not hold for this layer
            y = torch.empty((B, layer.OC, HO, WO), dtype=torch.int64, device=x.device)
            layer.forward(x, ws, padding, y_int64=y, out_f32=out)
    st = layer.stats(B, H, W, padding, ws)
    acts = layer.act_scales(B, H, W, padding, ws)
    rep = QuantReport(output=out, y_int=y, act_scale=float(acts[0]) if len(acts) == 1 else acts,
                      filter_scales=layer.filter_scales_native(),
                      saturations=st["saturations"] + layer.filter_saturations(),
                      values_quantized=st["values_quantized"])
    if report:
        # quant.cpp:282-291 on the device: fp64 output from the exact integer accumulator
        # against the exact int8 direct conv.
        out64 = torch.empty((B, layer.OC, HO, WO), dtype=torch.float64, device=x.device)
        layer.forward(x, ws, padding, out_f64=out64)
        w8 = as_int8_device(filters, "filters", x.device)
        ref = torch.empty((B, layer.OC, HO, WO), dtype=torch.int32, device=x.device)
        check(lib().sfc_direct_conv_int8(_ptr(x), B, C, H, W, _ptr(w8), layer.OC, spec.R, 1, padding, _ptr(ref),
                                         ctypes.c_void_p(_stream_ptr())))
        sums = (ctypes.c_double * 2)()
        check(lib().sfc_report_sq_err(_ptr(out64), _ptr(ref), out64.numel(), sums, ctypes.c_void_p(_stream_ptr())))
        err, sig = sums[0], sums[1]
        n = out64.numel()
        rep.mse = err / n
        rep.signal_energy = sig / n
        rep.snr_db = _snr_db(sig, err)
    return rep


def _quantized_fast_conv2d_real(input, filters, spec: AlgorithmSpec, padding: int, config: QuantConfig,
                                report: bool) -> QuantReport:
    """Real-valued tensors (the reference API's doubles): V, U, scales, vq / uq / pacc exactly
    as the reference computes them, the fp64 epilogue; output is float64 like DenseTensor."""
    x = as_f64_device(input)
    w = as_f64_device(filters, x.device)
    if x.dim() != 4 or w.dim() != 4:
        raise ValueError("conv2d expects 4-d NCHW tensors")
    if w.shape[1] != x.shape[1]:
        raise ValueError("input channel count does not match filters")
    B, C, H, W = x.shape
    if H + 2 * padding - spec.R + 1 <= 0 or W + 2 * padding - spec.R + 1 <= 0:
        raise ValueError("filter larger than padded input")
    layer = SfcLayer(spec, w, config.bits, config.filter_scope, config.search, act_scope=config.act_scope, real=True)
    HO, WO = H + 2 * padding - spec.R + 1, W + 2 * padding - spec.R + 1
    ws = layer.workspace(B, H, W, padding)
    out = torch.empty((B, layer.OC, HO, WO), dtype=torch.float64, device=x.device)
    layer.forward_f64(x, ws, padding, out_f64=out)
    st = layer.stats(B, H, W, padding, ws)
    acts = layer.act_scales(B, H, W, padding, ws)
    rep = QuantReport(output=out, y_int=None, act_scale=float(acts[0]) if len(acts) == 1 else acts,
                      filter_scales=layer.filter_scales_native(),
                      saturations=st["saturations"] + layer.filter_saturations(),
                      values_quantized=st["values_quantized"])
    if report:  # quant.cpp:282-291 against the fp64 direct conv (reference summation order)
        ref = torch.empty_like(out)
        check(lib().sfc_direct_conv_f64(_ptr(x), B, C, H, W, _ptr(w), layer.OC, spec.R, 1, padding, _ptr(ref),
                                        ctypes.c_void_p(_stream_ptr())))
        sums = (ctypes.c_double * 2)()
        check(lib().sfc_report_sq_err_f64(_ptr(out), _ptr(ref), out.numel(), sums, ctypes.c_void_p(_stream_ptr())))
        n = out.numel()
        rep.mse = sums[0] / n
        rep.signal_energy = sums[1] / n
        rep.snr_db = _snr_db(sums[1], sums[0])
    return rep


def fast_conv2d(input, filters, spec: AlgorithmSpec, padding: int = 0, reduced_products: bool = False) -> torch.Tensor:
    """conv.cpp:384-553 (the fp64 float path) on the device: fp64 NCHW output.  Returns the
    output tensor; fast_conv2d_counters() gives the product / tile counts.  reduced_products
    is FastConvOptions::reduced_products (the paired 6-for-9 block schedule)."""
    out, _ = fast_conv2d_counters(input, filters, spec, padding, reduced_products)
    return out


def fast_conv2d_counters(input, filters, spec: AlgorithmSpec, padding: int = 0, reduced_products: bool = False):
    x = as_f64_device(input)
    w = as_f64_device(filters, x.device)
    if x.dim() != 4 or w.dim() != 4:
        raise ValueError("conv2d expects 4-d NCHW tensors")
    if w.shape[1] != x.shape[1]:
        raise ValueError("input channel count does not match filters")
    if w.shape[2] != spec.R or w.shape[3] != spec.R:
        raise ValueError("filter size does not match algorithm")
    B, C, H, W = x.shape
    OC = w.shape[0]
    HO, WO = H + 2 * padding - spec.R + 1, W + 2 * padding - spec.R + 1
    if HO <= 0 or WO <= 0:
        raise ValueError("filter larger than padded input")
    out = torch.empty((B, OC, HO, WO), dtype=torch.float64, device=x.device)
    cnt = np.zeros(2, np.int64)
    check(lib().sfc_fast_conv_f64(ctypes.c_void_p(spec._handle), _ptr(x), B, C, H, W, _ptr(w), OC, padding,
                                  int(bool(reduced_products)), _ptr(out),
                                  cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.c_void_p(_stream_ptr())))
    return out, {"multiplications": int(cnt[0]), "tiles": int(cnt[1])}
