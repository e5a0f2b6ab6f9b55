// sfconv:: drop-in (B200 build) -- convolution entry points of the reference
// (include/sfconv/conv.hpp:12-36).  direct_conv2d and transform_filters run on
// the device for int8-valued tensors (exact int32 arithmetic); fast_conv2d, the
// reference's fp64 float path (conv.cpp:384-553), is not part of this build's
// device path yet and throws std::logic_error instead of falling back to a CPU.
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
