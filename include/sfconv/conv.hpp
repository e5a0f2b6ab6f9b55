// sfconv:: drop-in (B200 build) -- convolution entry points of the reference
// (include/sfconv/conv.hpp:12-36), all on the device.  direct_conv2d and
// transform_filters are exact int32 for int8-valued tensors and fp64 in the
// reference's summation order otherwise; fast_conv2d, the reference's fp64 float
// path (conv.cpp:384-553), forms V and U in the reference's order, contracts the
// K^2 frequencies (or the paired schedule's mults_reduced() slices when
// opts.reduced_products) as one batched fp64 GEMM and reports the counters.
// opts.threads is a host-CPU knob of the reference: accepted, without effect.
#pragma once

#include <cstdint>

#include "sfconv/spec.hpp"
#include "sfconv/tensor.hpp"

namespace sfconv {

struct ConvCounters {
    std::int64_t multiplications = 0;
    std::int64_t tiles = 0;
};

struct FastConvOptions {
    int threads = 1;
    bool reduced_products = false;
    ConvCounters* counters = nullptr;
};

DenseTensor direct_conv2d(const DenseTensor& input, const DenseTensor& filters, int stride = 1, int padding = 0);

DenseTensor transform_filters(const DenseTensor& filters, const AlgorithmSpec& spec);

DenseTensor fast_conv2d(const DenseTensor& input, const DenseTensor& filters, const AlgorithmSpec& spec,
                        int padding = 0, const FastConvOptions& opts = {});

}  // namespace sfconv
