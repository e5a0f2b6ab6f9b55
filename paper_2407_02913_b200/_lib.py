"""ctypes binding of libsfc_b200.so (the C-ABI declared in include/sfc_b200.h).

There is no fallback: if the shared library is missing or a call fails, this
module raises.  Error codes map onto the reference's exception classes:
SFC_ERR_INVALID / SFC_ERR_UNSUPPORTED -> ValueError (std::invalid_argument),
SFC_ERR_DOMAIN -> ArithmeticError (std::domain_error), SFC_ERR_CUDA -> RuntimeError.
"""
from __future__ import annotations

import ctypes
import os

# SFC_B200_LIB selects another in-tree build (the timeline build libsfc_b200_tl.so).
LIB_PATH = os.environ.get("SFC_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsfc_b200.so")

SFC_OK, SFC_ERR_INVALID, SFC_ERR_DOMAIN, SFC_ERR_UNSUPPORTED, SFC_ERR_CUDA = 0, -1, -2, -3, -4

# Every symbol include/sfc_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = (
    "sfc_last_error", "sfc_version", "sfc_catalog_json", "sfc_plan_create", "sfc_plan_destroy", "sfc_plan_dims",
    "sfc_plan_matrices", "sfc_layer_create", "sfc_layer_destroy", "sfc_layer_filter_scales",
    "sfc_layer_saturations", "sfc_layer_uq", "sfc_conv_workspace_size", "sfc_act_absmax", "sfc_conv_int8",
    "sfc_conv_int8_stages", "sfc_conv_forward", "sfc_conv_stats", "sfc_conv_views", "sfc_conv_schedule", "sfc_direct_conv_int8", "sfc_frequency_energy_int8",
    "sfc_transform_filters_int8", "sfc_debug_quantizer", "sfc_report_sq_err", "sfc_debug_timeline",
    "sfc_act_transform", "sfc_conv_kept", "sfc_layer_create_ex", "sfc_layer_filter_scales_native",
    "sfc_conv_act_scales", "sfc_layer_create_f64", "sfc_conv_forward_f64", "sfc_direct_conv_f64",
    "sfc_report_sq_err_f64", "sfc_fast_conv_f64", "sfc_transform_filters_f64",
    "sfc_general_prepare", "sfc_general_mse_partial", "sfc_general_conv",
)


class SfcError(RuntimeError):
    pass


class SfcInvalidArgument(ValueError):
    pass


class SfcUnsupported(SfcInvalidArgument):
    pass


class SfcDomainError(ArithmeticError):
    pass


class SfcCudaError(RuntimeError):
    pass


class Outputs(ctypes.Structure):
    _fields_ = [("y_int32", ctypes.c_void_p), ("y_int64", ctypes.c_void_p), ("out_f32", ctypes.c_void_p),
                ("out_f64", ctypes.c_void_p), ("out_i8", ctypes.c_void_p), ("requant_scale", ctypes.c_double)]


_lib = None

_vp = ctypes.c_void_p
_i = ctypes.c_int
_sz = ctypes.c_size_t
_i64p = ctypes.POINTER(ctypes.c_int64)

_SIGS = {
    "sfc_last_error": (ctypes.c_char_p, []),
    "sfc_version": (_i, []),
    "sfc_catalog_json": (_i, [ctypes.c_char_p, _sz, ctypes.POINTER(ctypes.c_uint64)]),
    "sfc_plan_create": (_i, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "sfc_plan_destroy": (_i, [_vp]),
    "sfc_plan_dims": (_i, [_vp, _i64p]),
    "sfc_plan_matrices": (_i, [_vp, _i64p, _i64p, _i64p]),
    "sfc_layer_create": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, ctypes.POINTER(_vp)]),
    "sfc_layer_destroy": (_i, [_vp]),
    "sfc_layer_filter_scales": (_i, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)]),
    "sfc_layer_saturations": (_i, [_vp, _i64p]),
    "sfc_layer_uq": (_i, [_vp, ctypes.POINTER(_vp), _i64p, _i64p]),
    "sfc_conv_workspace_size": (_i, [_vp, _i, _i, _i, _i, ctypes.POINTER(_sz)]),
    "sfc_act_absmax": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "sfc_conv_int8": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp, _sz, ctypes.POINTER(Outputs), _vp]),
    "sfc_conv_int8_stages": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp, _sz, ctypes.POINTER(Outputs), ctypes.c_uint, _vp]),
    "sfc_conv_forward": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _sz, ctypes.POINTER(Outputs), _vp]),
    "sfc_general_prepare": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _sz, ctypes.POINTER(_vp), ctypes.POINTER(_i), _vp]),
    "sfc_general_mse_partial": (_i, [_vp, _i, _i, _i, _i, _vp, _sz, _vp, _vp, _vp]),
    "sfc_general_conv": (_i, [_vp, _i, _i, _i, _i, _vp, _sz, _vp, ctypes.POINTER(Outputs), _vp]),
    "sfc_act_transform": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp, _sz, _vp]),
    "sfc_layer_create_ex": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _i, _vp, ctypes.POINTER(_vp)]),
    "sfc_layer_filter_scales_native": (_i, [_vp, _vp, _i64p]),
    "sfc_conv_act_scales": (_i, [_vp, _i, _i, _i, _i, _vp, _sz, _vp, _i64p, _vp]),
    "sfc_layer_create_f64": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _i, _vp, ctypes.POINTER(_vp)]),
    "sfc_conv_forward_f64": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _sz, ctypes.POINTER(Outputs), _vp]),
    "sfc_direct_conv_f64": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _vp, _vp]),
    "sfc_report_sq_err_f64": (_i, [_vp, _vp, ctypes.c_int64, ctypes.POINTER(ctypes.c_double), _vp]),
    "sfc_fast_conv_f64": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _i, _i, _i, _vp, _i64p, _vp]),
    "sfc_conv_kept": (_i, [_vp, _i, _i, _i, _i, _vp, _vp, _sz, ctypes.POINTER(Outputs), _vp]),
    "sfc_conv_stats": (_i, [_vp, _i, _i, _i, _i, _vp, _sz, _i64p, _vp]),
    "sfc_conv_views": (_i, [_vp, _i, _i, _i, _i, _vp, _sz, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64p]),
    "sfc_conv_schedule": (_i, [_vp, _i, _i, _i, _i, ctypes.POINTER(_i)]),
    "sfc_direct_conv_int8": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _vp, _vp]),
    "sfc_frequency_energy_int8": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _vp]),
    "sfc_transform_filters_int8": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "sfc_transform_filters_f64": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "sfc_debug_quantizer": (_i, [_i, _i, _vp, _i64p, _vp]),
    "sfc_debug_timeline": (_i, [_vp, _i]),
    "sfc_report_sq_err": (_i, [_vp, _vp, ctypes.c_int64, ctypes.POINTER(ctypes.c_double), _vp]),
}


def lib():
    """Load libsfc_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SfcError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc == SFC_OK:
        return
    msg = lib().sfc_last_error().decode(errors="replace")
    if rc == SFC_ERR_UNSUPPORTED:
        raise SfcUnsupported(msg)
    if rc == SFC_ERR_INVALID:
        raise SfcInvalidArgument(msg)
    if rc == SFC_ERR_DOMAIN:
        raise SfcDomainError(msg)
    raise SfcCudaError(msg)
