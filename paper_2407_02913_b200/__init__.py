"""B200-native quantized SFC 3x3 convolution (Symbolic Fourier Convolution, arXiv 2407.02913).

The compute path is libsfc_b200.so (hand-written sm_100a CUDA behind the C-ABI in
include/sfc_b200.h); this package is the Python host mirror of the reference's
sfconv:: interface (proj/include/sfconv/*.hpp).  There is no CPU fallback.
"""
from .sfconv import (ActScaleScope, AlgorithmSpec, FilterScaleScope, QuantConfig, QuantReport, ScaleSearch,  # noqa
                     SfcLayer, catalog_algorithm, catalog_export_json, catalog_names, direct_conv2d,
                     fast_conv2d, fast_conv2d_counters, frequency_energy, quantize_value, quantized_fast_conv2d, scale_minmax, scale_mse_grid,
                     transform_filters)

__all__ = ["ActScaleScope", "AlgorithmSpec", "FilterScaleScope", "QuantConfig", "QuantReport", "ScaleSearch",
           "SfcLayer", "catalog_algorithm", "catalog_export_json", "catalog_names", "direct_conv2d",
           "fast_conv2d", "fast_conv2d_counters", "frequency_energy", "quantize_value", "quantized_fast_conv2d", "scale_minmax", "scale_mse_grid",
           "transform_filters"]
