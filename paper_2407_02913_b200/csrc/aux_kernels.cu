// Offline filter stage and the report / API kernels.
//   k_filter_prepare     U = G f G^T (R x R filters), per-oc minmax scale, exact RNE quantize into the
//                        GEMM B operand uq[f][oc][ic]   (conv.cpp:352-382, quant.cpp:183-229)
//   k_direct_conv        exact int8 correlation (int32)  (conv.cpp:320-350, quant.cpp:282)
//   k_freq_energy        sum of V^2 per frequency, exact (quant.cpp:136-150)
//   k_transform_filters  U as int32                      (conv.cpp:352-382)
#include <cstdlib>

#include <cuda_runtime.h>

#include "common.cuh"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"

namespace sfcb200 {

// Row k of U = G f G^T for one R x R filter: U[k][l] = sum_j (sum_r G[k][r] f[r][j]) G[l][j].
template <int V, class Fn>
__device__ __forceinline__ void filter_rows(const int (&f)[Tab<V>::R][Tab<V>::R], Fn&& fn) {
    using T = Tab<V>;
    constexpr int R = T::R;
#pragma unroll
    for (int k = 0; k < T::K; ++k) {
        int tmp[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            int acc = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) acc += T::g(k, r) * f[r][j];
            tmp[j] = acc;
        }
#pragma unroll
        for (int l = 0; l < T::K; ++l) {
            int acc = 0;
#pragma unroll
            for (int j = 0; j < R; ++j) acc += tmp[j] * T::g(l, j);
            fn(k, l, acc);
        }
    }
}

template <int R>
__device__ __forceinline__ void load_filter(const int8_t* __restrict__ w, size_t base, int (&f)[R][R]) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < R; ++c) f[r][c] = w[base + r * R + c];
}

template <int V>
__global__ void __launch_bounds__(128) k_filter_prepare(const int8_t* __restrict__ w, int OC, int IC, int Cpad,
                                                        int OCpad, int bits, double* __restrict__ sf_out,
                                                        int* __restrict__ umax_out, int8_t* __restrict__ uqB,
                                                        unsigned long long* sat) {
    using T = Tab<V>;
    const int oc = blockIdx.x;
    const int qmax = (1 << (bits - 1)) - 1;
    __shared__ int s_max[4];
    int local = 0;
    for (int ic = threadIdx.x; ic < IC; ic += blockDim.x) {
        int f[T::R][T::R];
        load_filter<T::R>(w, (size_t(oc) * IC + ic) * T::R * T::R, f);
        filter_rows<V>(f, [&](int, int, int u) { local = max(local, abs(u)); });
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = local;
    __syncthreads();
    const int umax = max(max(s_max[0], s_max[1]), max(s_max[2], s_max[3]));
    const double sf = fmax(double(umax) / double(qmax), 1e-8);  // scale_minmax, quant.cpp:117-120
    if (threadIdx.x == 0) {
        sf_out[oc] = sf;
        if (umax_out) umax_out[oc] = umax;
    }
    for (int ic = threadIdx.x; ic < IC; ic += blockDim.x) {
        int f[T::R][T::R];
        load_filter<T::R>(w, (size_t(oc) * IC + ic) * T::R * T::R, f);
        filter_rows<V>(f, [&](int k, int l, int u) {
            const int q = clamp_q(exact_q(u, sf), qmax, sat);
            uqB[(size_t(k * T::K + l) * OCpad + oc) * Cpad + ic] = int8_t(q);
        });
    }
}

__global__ void __launch_bounds__(256) k_direct_conv(const int8_t* __restrict__ x, int B, int C, int H, int W,
                                                     const int8_t* __restrict__ w, int OC, int R, int stride, int pad,
                                                     int HO, int WO, int32_t* __restrict__ out) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)B * OC * HO * WO) return;
    const int ow = int(idx % WO), oh = int((idx / WO) % HO), oc = int((idx / ((long long)WO * HO)) % OC);
    const int b = int(idx / ((long long)WO * HO * OC));
    int acc = 0;
    for (int ic = 0; ic < C; ++ic)
        for (int fr = 0; fr < R; ++fr) {
            const int ih = oh * stride - pad + fr;
            if (ih < 0 || ih >= H) continue;
            for (int fc = 0; fc < R; ++fc) {
                const int iw = ow * stride - pad + fc;
                if (iw < 0 || iw >= W) continue;
                acc += int(x[((size_t(b) * C + ic) * H + ih) * W + iw]) *
                       int(w[((size_t(oc) * C + ic) * R + fr) * R + fc]);
            }
        }
    out[idx] = acc;
}

template <int V>
__global__ void __launch_bounds__(256) k_freq_energy(const int8_t* __restrict__ x, ConvGeom g,
                                                     unsigned long long* __restrict__ sum) {
    using T = Tab<V>;
    __shared__ unsigned long long s_sum[T::F];
    for (int i = threadIdx.x; i < T::F; i += blockDim.x) s_sum[i] = 0;
    __syncthreads();
    const long long n_items = (long long)g.T * g.C;
    for (long long item = (long long)blockIdx.x * blockDim.x + threadIdx.x; item < n_items;
         item += (long long)gridDim.x * blockDim.x) {
        const int c = int(item % g.C);
        const int t = int(item / g.C);
        const int per_img = g.th * g.tw;
        const int b = t / per_img, ti = (t % per_img) / g.tw, tj = t % g.tw;
        int xw[T::n][T::n];
#pragma unroll
        for (int r = 0; r < T::n; ++r)
#pragma unroll
            for (int s = 0; s < T::n; ++s) {
                const int ih = ti * T::M - g.pad + r, iw = tj * T::M - g.pad + s;
                xw[r][s] = (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
                               ? int(x[((size_t(b) * g.C + c) * g.H + ih) * g.W + iw])
                               : 0;
            }
#pragma unroll
        for (int k = 0; k < T::K; ++k) {
            int row[T::n];
#pragma unroll
            for (int s = 0; s < T::n; ++s) {
                int acc = 0;
#pragma unroll
                for (int r = 0; r < T::n; ++r) acc += T::bt(k, r) * xw[r][s];
                row[s] = acc;
            }
#pragma unroll
            for (int l = 0; l < T::K; ++l) {
                int v = 0;
#pragma unroll
                for (int s = 0; s < T::n; ++s) v += row[s] * T::bt(l, s);
                atomicAdd(&s_sum[k * T::K + l], (unsigned long long)((long long)v * v));
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < T::F; i += blockDim.x)
        if (s_sum[i]) atomicAdd(&sum[i], s_sum[i]);
}

template <int V>
__global__ void __launch_bounds__(128) k_transform_filters(const int8_t* __restrict__ w, int OC, int IC,
                                                           int32_t* __restrict__ u) {
    using T = Tab<V>;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)OC * IC) return;
    int f[T::R][T::R];
    load_filter<T::R>(w, size_t(idx) * T::R * T::R, f);
    filter_rows<V>(f, [&](int k, int l, int v) { u[idx * T::F + k * T::K + l] = v; });
}

// ============================================================================ host
cudaError_t launch_filter_prepare(int variant, const int8_t* w, int OC, int IC, int Cpad, int OCpad, int bits,
                                  double* sf, int* umax, int8_t* uqB, unsigned long long* sat, cudaStream_t st) {
    switch (variant) {
        case 0: k_filter_prepare<0><<<OC, 128, 0, st>>>(w, OC, IC, Cpad, OCpad, bits, sf, umax, uqB, sat); break;
        case 1: k_filter_prepare<1><<<OC, 128, 0, st>>>(w, OC, IC, Cpad, OCpad, bits, sf, umax, uqB, sat); break;
        case 2: k_filter_prepare<2><<<OC, 128, 0, st>>>(w, OC, IC, Cpad, OCpad, bits, sf, umax, uqB, sat); break;
        case 3: k_filter_prepare<3><<<OC, 128, 0, st>>>(w, OC, IC, Cpad, OCpad, bits, sf, umax, uqB, sat); break;
        default: k_filter_prepare<4><<<OC, 128, 0, st>>>(w, OC, IC, Cpad, OCpad, bits, sf, umax, uqB, sat); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_direct_conv(const int8_t* x, int B, int C, int H, int W, const int8_t* w, int OC, int R,
                               int stride, int pad, int32_t* out, cudaStream_t st) {
    const int HO = (H + 2 * pad - R) / stride + 1, WO = (W + 2 * pad - R) / stride + 1;
    const long long n = (long long)B * OC * HO * WO;
    k_direct_conv<<<int((n + 255) / 256), 256, 0, st>>>(x, B, C, H, W, w, OC, R, stride, pad, HO, WO, out);
    return cudaGetLastError();
}

cudaError_t launch_freq_energy(int variant, const int8_t* x, const ConvGeom& g, unsigned long long* sum,
                               cudaStream_t st) {
    const long long n = (long long)g.T * g.C;
    int blocks = int((n + 255) / 256);
    blocks = blocks > 4 * 148 ? 4 * 148 : (blocks < 1 ? 1 : blocks);
    switch (variant) {
        case 0: k_freq_energy<0><<<blocks, 256, 0, st>>>(x, g, sum); break;
        case 1: k_freq_energy<1><<<blocks, 256, 0, st>>>(x, g, sum); break;
        case 2: k_freq_energy<2><<<blocks, 256, 0, st>>>(x, g, sum); break;
        case 3: k_freq_energy<3><<<blocks, 256, 0, st>>>(x, g, sum); break;
        default: k_freq_energy<4><<<blocks, 256, 0, st>>>(x, g, sum); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_transform_filters(int variant, const int8_t* w, int OC, int IC, int32_t* u, cudaStream_t st) {
    const long long n = (long long)OC * IC;
    const int blocks = int((n + 127) / 128);
    switch (variant) {
        case 0: k_transform_filters<0><<<blocks, 128, 0, st>>>(w, OC, IC, u); break;
        case 1: k_transform_filters<1><<<blocks, 128, 0, st>>>(w, OC, IC, u); break;
        case 2: k_transform_filters<2><<<blocks, 128, 0, st>>>(w, OC, IC, u); break;
        case 3: k_transform_filters<3><<<blocks, 128, 0, st>>>(w, OC, IC, u); break;
        default: k_transform_filters<4><<<blocks, 128, 0, st>>>(w, OC, IC, u); break;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- geometry
void geom_init(ConvGeom& g, int variant, int B, int C, int H, int W, int pad, int OC) {
    static constexpr int kM[5] = {Tab<0>::M, Tab<1>::M, Tab<2>::M, Tab<3>::M, Tab<4>::M};
    static constexpr int kR[5] = {Tab<0>::R, Tab<1>::R, Tab<2>::R, Tab<3>::R, Tab<4>::R};
    const int M = kM[variant], R = kR[variant];
    g.B = B, g.C = C, g.H = H, g.W = W, g.pad = pad, g.OC = OC;
    g.HO = H + 2 * pad - R + 1;
    g.WO = W + 2 * pad - R + 1;
    g.th = (g.HO + M - 1) / M;
    g.tw = (g.WO + M - 1) / M;
    g.T = B * g.th * g.tw;
    g.Tpad = (g.T + kRowsPerTile - 1) / kRowsPerTile * kRowsPerTile;
    g.BK = C > 64 ? 128 : 64;
    g.Cpad = (C + g.BK - 1) / g.BK * g.BK;
    g.BN = OC <= 64 ? 64 : (OC <= 128 ? 128 : 256);
    if (const char* e = std::getenv("SFC_BN_MAX")) {  // experiment knob: cap the GEMM N tile (64 / 128)
        const int cap = std::atoi(e);
        if ((cap == 64 || cap == 128) && g.BN > cap && OC > 256) g.BN = cap;
    }
    g.OCpad = (OC + g.BN - 1) / g.BN * g.BN;
    g.row0 = 0;
    g.nrows = B * g.th;
    g.p24 = 0;
    g.p2s = 0;
}

PChunk p_chunk(const ConvGeom& g, int F) {
    size_t budget = 0;  // opt-in (see sfc_kernels.hpp)
    if (const char* e = std::getenv("SFC_PCHUNK_MB")) budget = size_t(std::atol(e)) << 20;
    const size_t per_row = size_t(F) * g.OCpad * 4;  // P bytes per tile
    const int rows_total = g.B * g.th;
    if (budget == 0 || per_row * g.Tpad <= budget) return PChunk{rows_total, g.Tpad, 1};
    size_t max_tiles = budget / per_row / kRowsPerTile * kRowsPerTile;
    if (max_tiles < size_t(kRowsPerTile)) max_tiles = kRowsPerTile;
    int rows_max = int(max_tiles / size_t(g.tw));
    if (rows_max < 1) rows_max = 1;
    const int n = (rows_total + rows_max - 1) / rows_max;
    const int rows = (rows_total + n - 1) / n;  // balanced chunks
    const int tcpad = (rows * g.tw + kRowsPerTile - 1) / kRowsPerTile * kRowsPerTile;
    return PChunk{rows, tcpad, (rows_total + rows - 1) / rows};
}

size_t workspace_bytes(const ConvGeom& g, int F) {
    auto up = [](size_t v) { return (v + 255) / 256 * 256; };
    return up(kWsHeader) + up(size_t(F) * g.Tpad * g.Cpad) + up(size_t(F) * p_chunk(g, F).tcpad * g.OCpad * 4) +
           up(size_t(F) * g.Tpad * g.Cpad * 2);  // kept int16 V
}

}  // namespace sfcb200

namespace sfcb200 {
// Report sums for quantized_fast_conv2d (quant.cpp:283-291): sums[0] += sum (out - ref)^2,
// sums[1] += sum ref^2 in fp64 (ref is the exact int8 direct conv).
template <class TR>
__global__ void __launch_bounds__(256) k_sq_err(const double* __restrict__ out, const TR* __restrict__ ref,
                                                long long n, double* __restrict__ sums) {
    double e = 0.0, s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double r = double(ref[i]), d = out[i] - r;
        e += d * d;
        s += r * r;
    }
    __shared__ double se[8], ss[8];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, o);
        s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if ((threadIdx.x & 31) == 0) se[threadIdx.x >> 5] = e, ss[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {  // per-block partials; k_sum_partials adds them in block order
        double a = 0.0, b = 0.0;
        for (int w = 0; w < 8; ++w) a += se[w], b += ss[w];
        sums[2 + 2 * blockIdx.x] = a;
        sums[3 + 2 * blockIdx.x] = b;
    }
}

// sums[0..1] = the block partials summed in a fixed order: the report is bitwise
// repeatable (the grid size depends on n only).
__global__ void k_sum_partials(double* __restrict__ sums, int blocks) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < blocks; ++i) a += sums[2 + 2 * i], b += sums[3 + 2 * i];
    sums[0] = a;
    sums[1] = b;
}

__global__ void k_zero_words(uint32_t* __restrict__ p, int words) {
    tl_mark(kTlZero, 0);
    griddep_wait();
    tl_mark(kTlZero, 1);
    griddep_launch_dependents();
    if (int(threadIdx.x) < words) p[threadIdx.x] = 0u;
    tl_mark(kTlZero, 2);
}

SFC_TL_UNIT_READER(tl_read_aux)

cudaError_t launch_zero_words(uint32_t* p, int words, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_zero_words, p, words);
}

cudaError_t launch_sq_err(const double* out, const int32_t* ref, long long n, double* sums, cudaStream_t st) {
    long long blocks = (n + 255) / 256;
    blocks = blocks > kSqErrBlocks ? kSqErrBlocks : (blocks < 1 ? 1 : blocks);
    k_sq_err<int32_t><<<int(blocks), 256, 0, st>>>(out, ref, n, sums);
    k_sum_partials<<<1, 1, 0, st>>>(sums, int(blocks));
    return cudaGetLastError();
}

cudaError_t launch_sq_err_f64(const double* out, const double* ref, long long n, double* sums, cudaStream_t st) {
    long long blocks = (n + 255) / 256;
    blocks = blocks > kSqErrBlocks ? kSqErrBlocks : (blocks < 1 ? 1 : blocks);
    k_sq_err<double><<<int(blocks), 256, 0, st>>>(out, ref, n, sums);
    k_sum_partials<<<1, 1, 0, st>>>(sums, int(blocks));
    return cudaGetLastError();
}
}  // namespace sfcb200
