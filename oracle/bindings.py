"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU oracle and the compiled reference.

* ``liboracle``  -- our C restatement (oracle/sfc_oracle.c), always built.
* ``libref``     -- the unmodified reference (oracle/_ref/libsfconv_ref.so), built
                    from /root/reference/proj/src by oracle/Makefile where that tree
                    exists; the .so travels to the GPU box with the repo snapshot.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsfconv_ref.so")

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_i8p = ctypes.POINTER(ctypes.c_int8)


class SfoConfig(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_int), ("act_scope", ctypes.c_int), ("filter_scope", ctypes.c_int),
                ("search", ctypes.c_int), ("threads", ctypes.c_int), ("want_report", ctypes.c_int),
                ("vmax_override", ctypes.c_int64), ("act_scale_override", ctypes.POINTER(ctypes.c_double))]


class SfoReport(ctypes.Structure):
    _fields_ = [("mse", ctypes.c_double), ("signal_energy", ctypes.c_double), ("snr_db", ctypes.c_double),
                ("saturations", ctypes.c_int64), ("values_quantized", ctypes.c_int64),
                ("vmax", ctypes.c_int64), ("tiles", ctypes.c_int64),
                ("th", ctypes.c_int), ("tw", ctypes.c_int), ("HO", ctypes.c_int), ("WO", ctypes.c_int)]


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _oracle = ctypes.CDLL(ORACLE_SO)
        _oracle.sfo_last_error.restype = ctypes.c_char_p
        _oracle.sfo_quantize_value.restype = ctypes.c_int64
        _oracle.sfo_quantize_value.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int, _i64p]
        _oracle.sfo_scale_minmax.restype = ctypes.c_double
        _oracle.sfo_scale_minmax.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int]
        _oracle.sfo_scale_mse_grid.restype = ctypes.c_double
        _oracle.sfo_scale_mse_grid.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int]
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        _ref = ctypes.CDLL(REF_SO)
        _ref.ref_last_error.restype = ctypes.c_char_p
        _ref.ref_quantize_value.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int, _i64p, _i64p]
        _ref.ref_scale.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _f64p]
    return _ref


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _check(lib, rc, which):
    if rc != 0:
        err = (lib.sfo_last_error() if which == "oracle" else lib.ref_last_error()).decode()
        exc = ValueError if rc == -1 else RuntimeError
        raise exc(err)


# ----------------------------------------------------------------------------- specs
def spec(name: str, source: str = "oracle") -> dict:
    dims = np.zeros(10, np.int64)
    bt = np.zeros(16 * 16, np.int64)  # room for every catalogued SFC size (K <= 14, n <= 10, R <= 7)
    g = np.zeros(16 * 8, np.int64)
    a = np.zeros(16 * 8, np.int64)
    if source == "oracle":
        lib = oracle_lib()
        _check(lib, lib.sfo_spec(name.encode(), _ptr(dims, _i64p), _ptr(bt, _i64p), _ptr(g, _i64p),
                                 _ptr(a, _i64p)), "oracle")
    else:
        lib = ref_lib()
        _check(lib, lib.ref_spec(name.encode(), _ptr(dims, _i64p), _ptr(bt, _i64p), _ptr(g, _i64p),
                                 _ptr(a, _i64p)), "ref")
    K, n, M, R = (int(v) for v in dims[:4])
    return dict(name=name, K=K, n=n, M=M, R=R, N=int(dims[4]), offset=int(dims[5]), a_denom=int(dims[6]),
                n_corrections=int(dims[7]), mults_full=int(dims[8]), mults_reduced=int(dims[9]),
                BT=bt[:K * n].reshape(K, n).copy(), G=g[:K * R].reshape(K, R).copy(),
                A=a[:K * M].reshape(K, M).copy())


# ----------------------------------------------------------------------------- oracle
def quantize_value(v: float, scale: float, bits: int):
    sat = ctypes.c_int64(0)
    q = oracle_lib().sfo_quantize_value(v, scale, bits, ctypes.byref(sat))
    return q, sat.value


def scale_minmax(vals, bits):
    v = np.ascontiguousarray(vals, np.float64)
    return oracle_lib().sfo_scale_minmax(_ptr(v, _f64p), v.size, bits)


def scale_mse_grid(vals, bits):
    v = np.ascontiguousarray(vals, np.float64)
    return oracle_lib().sfo_scale_mse_grid(_ptr(v, _f64p), v.size, bits)


def quantized_conv(x: np.ndarray, w: np.ndarray, spec_name: str, pad: int = 1, bits: int = 8,
                   act_scope: int = 0, filter_scope: int = 0, search: int = 0, threads: int | None = None,
                   want=("out", "y_int"), report: bool = False, vmax_override: int = -1,
                   act_scale_override=None) -> dict:
    """Run the C restatement.  x: int8 [B,C,H,W], w: int8 [OC,C,R,R].  act_scale_override: the
    activation scales (1 or F) to quantize with (a batch shard with the full batch's scales)."""
    lib = oracle_lib()
    x = np.ascontiguousarray(x, np.int8)
    w = np.ascontiguousarray(w, np.int8)
    B, C, H, W = x.shape
    OC = w.shape[0]
    sp = spec(spec_name)
    K, M, R = sp["K"], sp["M"], sp["R"]
    F = K * K
    if w.shape[1:] != (C, R, R):
        raise ValueError("filter shape does not match algorithm")
    HO, WO = H + 2 * pad - R + 1, W + 2 * pad - R + 1
    th, tw = -(-HO // M), -(-WO // M)
    T = B * th * tw
    res = {}
    out = np.empty((B, OC, HO, WO), np.float64) if ("out" in want or report) else None
    y = np.empty((B, OC, HO, WO), np.int64) if "y_int" in want else None
    pacc = np.empty((T, OC, F), np.int64) if "pacc" in want else None
    vq = np.empty((T, C, F), np.int32) if "vq" in want else None
    uq = np.empty((OC, C, F), np.int32) if "uq" in want else None
    act = np.empty(F, np.float64)
    fil = np.empty(OC * F, np.float64)
    aso = None if act_scale_override is None else np.ascontiguousarray(act_scale_override, np.float64)
    cfg = SfoConfig(bits, act_scope, filter_scope, search, threads or os.cpu_count() or 1, int(report),
                    int(vmax_override), None if aso is None else _ptr(aso, _f64p))
    rep = SfoReport()
    rc = lib.sfo_quantized_conv(_ptr(x, _i8p), B, C, H, W, _ptr(w, _i8p), OC, spec_name.encode(), pad,
                                ctypes.byref(cfg), _ptr(out, _f64p), _ptr(y, _i64p), _ptr(pacc, _i64p),
                                _ptr(vq, _i32p), _ptr(uq, _i32p), _ptr(act, _f64p), _ptr(fil, _f64p),
                                ctypes.byref(rep))
    _check(lib, rc, "oracle")
    for k, v in (("out", out), ("y_int", y), ("pacc", pacc), ("vq", vq), ("uq", uq)):
        if v is not None:
            res[k] = v
    res["act_scale"] = act[: (1 if act_scope == 0 else F)].copy()
    res["fil_scale"] = fil[: {0: OC, 1: F, 2: OC * F}[filter_scope]].copy()
    res["report"] = {f: getattr(rep, f) for f, _ in SfoReport._fields_}
    res["spec"] = sp
    return res


def direct_conv(x, w, pad=1):
    lib = oracle_lib()
    x = np.ascontiguousarray(x, np.int8)
    w = np.ascontiguousarray(w, np.int8)
    B, C, H, W = x.shape
    OC, _, R, _ = w.shape
    out = np.empty((B, OC, H + 2 * pad - R + 1, W + 2 * pad - R + 1), np.float64)
    _check(lib, lib.sfo_direct_conv(_ptr(x, _i8p), B, C, H, W, _ptr(w, _i8p), OC, R, pad, 1,
                                    _ptr(out, _f64p)), "oracle")
    return out


def execute_tile(spec_name, x, f):
    lib = oracle_lib()
    sp = spec(spec_name)
    x = np.ascontiguousarray(x, np.int64)
    f = np.ascontiguousarray(f, np.int64)
    y = np.empty((sp["M"], sp["M"]), np.int64)
    _check(lib, lib.sfo_execute_tile(spec_name.encode(), _ptr(x, _i64p), _ptr(f, _i64p), _ptr(y, _i64p)),
           "oracle")
    return y


def check_identity(spec_name):
    return oracle_lib().sfo_check_identity(spec_name.encode())


# ----------------------------------------------------------------------------- reference
def ref_quantized_fast_conv2d(x, w, spec_name, pad=1, bits=8, act_scope=0, filter_scope=0, search=0):
    lib = ref_lib()
    xd = np.ascontiguousarray(x, np.float64)
    wd = np.ascontiguousarray(w, np.float64)
    B, C, H, W = xd.shape
    OC, IC, R, _ = wd.shape
    out = np.empty((B, OC, H + 2 * pad - R + 1, W + 2 * pad - R + 1), np.float64)
    rep = np.zeros(5, np.float64)
    rc = lib.ref_quantized_fast_conv2d(_ptr(xd, _f64p), B, C, H, W, _ptr(wd, _f64p), OC, IC, R,
                                       spec_name.encode(), pad, bits, act_scope, filter_scope, search,
                                       _ptr(out, _f64p), _ptr(rep, _f64p))
    _check(lib, rc, "ref")
    return out, dict(mse=rep[0], signal_energy=rep[1], snr_db=rep[2], saturations=int(rep[3]),
                     values_quantized=int(rep[4]))


def ref_quantize_value(v, scale, bits):
    lib = ref_lib()
    sat, q = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib, lib.ref_quantize_value(v, scale, bits, ctypes.byref(sat), ctypes.byref(q)), "ref")
    return q.value, sat.value


def ref_scale(vals, bits, mse_grid=False):
    lib = ref_lib()
    v = np.ascontiguousarray(vals, np.float64)
    out = ctypes.c_double(0)
    _check(lib, lib.ref_scale(_ptr(v, _f64p), v.size, bits, int(mse_grid), ctypes.byref(out)), "ref")
    return out.value


def ref_catalog_json():
    lib = ref_lib()
    buf = ctypes.create_string_buffer(1 << 20)
    h = ctypes.c_uint64(0)
    _check(lib, lib.ref_catalog_json(buf, 1 << 20, ctypes.byref(h)), "ref")
    return buf.value.decode(), h.value


def ref_transform_filters(w, spec_name):
    lib = ref_lib()
    wd = np.ascontiguousarray(w, np.float64)
    OC, IC, R, _ = wd.shape
    K = spec(spec_name)["K"]
    out = np.empty((OC, IC, K, K), np.float64)
    _check(lib, lib.ref_transform_filters(_ptr(wd, _f64p), OC, IC, R, spec_name.encode(), _ptr(out, _f64p)),
           "ref")
    return out


def ref_direct_conv2d(x, w, pad=1, stride=1):
    lib = ref_lib()
    xd = np.ascontiguousarray(x, np.float64)
    wd = np.ascontiguousarray(w, np.float64)
    B, C, H, W = xd.shape
    OC, IC, R, _ = wd.shape
    HO = (H + 2 * pad - R) // stride + 1
    WO = (W + 2 * pad - R) // stride + 1
    out = np.empty((B, OC, HO, WO), np.float64)
    _check(lib, lib.ref_direct_conv2d(_ptr(xd, _f64p), B, C, H, W, _ptr(wd, _f64p), OC, IC, R, stride, pad,
                                      _ptr(out, _f64p)), "ref")
    return out


def ref_fast_conv2d(x, w, spec_name, pad=1, threads=1, reduced=False):
    lib = ref_lib()
    xd = np.ascontiguousarray(x, np.float64)
    wd = np.ascontiguousarray(w, np.float64)
    B, C, H, W = xd.shape
    OC, IC, R, _ = wd.shape
    out = np.empty((B, OC, H + 2 * pad - R + 1, W + 2 * pad - R + 1), np.float64)
    mults = np.zeros(2, np.int64)
    _check(lib, lib.ref_fast_conv2d(_ptr(xd, _f64p), B, C, H, W, _ptr(wd, _f64p), OC, IC, R,
                                    spec_name.encode(), pad, threads, int(reduced), _ptr(out, _f64p),
                                    _ptr(mults, _i64p)), "ref")
    return out, mults


def ref_frequency_energy(x, spec_name, pad=0):
    lib = ref_lib()
    xd = np.ascontiguousarray(x, np.float64)
    B, C, H, W = xd.shape
    K = spec(spec_name)["K"]
    e = np.empty(K * K, np.float64)
    _check(lib, lib.ref_frequency_energy(_ptr(xd, _f64p), B, C, H, W, spec_name.encode(), pad, _ptr(e, _f64p)),
           "ref")
    return e


def ref_execute_tile(spec_name, x, f):
    lib = ref_lib()
    sp = spec(spec_name, "ref")
    x = np.ascontiguousarray(x, np.int64)
    f = np.ascontiguousarray(f, np.int64)
    y = np.empty((sp["M"], sp["M"]), np.int64)
    _check(lib, lib.ref_execute_tile_exact(spec_name.encode(), _ptr(x, _i64p), _ptr(f, _i64p), _ptr(y, _i64p)),
           "ref")
    return y
