// Non-default QuantConfig on the device: per-frequency activation
// scales, per-frequency / per-(channel, frequency) filter scales and the MseGrid scale
// search (quant.cpp:13-30, 117-134, 163-229, 242-263).
//
// Scale search follows the reference bit for bit: a group's MinMax scale is
// max(absmax / qmax, 1e-8); MseGrid evaluates quant_group_mse for the MinMax scale and 100
// grid candidates, each as ONE sequential fp64 sum over the group's values in the
// reference's order, with the reference's rounding steps (__ddiv_rn / __dmul_rn / __dsub_rn /
// __dadd_rn: no FMA contraction, like the reference's x86-64 build), and keeps the first
// strict minimum.  Candidates run as the lanes of a warp so every value load is a broadcast.
// Quantization here is the reference's fp64 nearbyint(v / s) with clamping and saturation
// counting (these configurations are parity paths, not the tuned default).
#include <cuda_runtime.h>

#include "common.cuh"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"

namespace sfcb200 {

namespace {
constexpr int kCands = 101;  // the MinMax scale + 100 grid points (quant.cpp:125-131)

__device__ __forceinline__ double grid_scale(double base, int cand) {  // cand 0 = base
    if (cand == 0) return base;
    const double t = __dadd_rn(0.3, __ddiv_rn(__dmul_rn(0.7, double(cand - 1)), 99.0));
    return fmax(__dmul_rn(base, t), 1e-8);
}

__device__ __forceinline__ double mse_term(double v, double s, double qmax, double qmin) {
    double q = rint(__ddiv_rn(v, s));
    q = fmin(qmax, fmax(qmin, q));
    const double d = __dsub_rn(v, __dmul_rn(q, s));
    return __dmul_rn(d, d);
}

// Group g of the transformed filters U[oc][ic][f] (int32, exact) for a filter scope:
// base offset, element stride and count, in the reference's value order (quant.cpp:193-219).
struct FilGroup {
    long long base, stride, count;
};
__device__ __forceinline__ FilGroup fil_group(int scope, int g, int OC, int IC, int F) {
    if (scope == 0) return {(long long)g * IC * F, 1, (long long)IC * F};   // PerChannel: (ic, f)
    if (scope == 1) return {g, F, (long long)OC * IC};                       // PerFrequency: (oc, ic)
    return {(long long)(g / F) * IC * F + g % F, F, IC};                     // PerChannelFrequency: ic
}
}  // namespace

// One warp per group, lane = candidate chunk: absmax (exact, order-free), then for
// MseGrid the 101 candidate errors (lanes 0..31 take candidates lane, lane+32, ...).
// err_out[g * kCands + cand]; scale_out[g] is the MinMax scale (the MseGrid pick follows).
template <class TU>
__global__ void __launch_bounds__(32) k_fil_scales(const TU* __restrict__ U, int OC, int IC, int F, int scope,
                                                   int mse, int bits, double* __restrict__ scale_out,
                                                   double* __restrict__ err_out) {
    const int g = blockIdx.x, lane = threadIdx.x;
    const FilGroup G = fil_group(scope, g, OC, IC, F);
    double amax = 0.0;  // exact and order-free (group_absmax, quant.cpp:13-17)
    for (long long i = lane; i < G.count; i += 32) amax = fmax(amax, fabs(double(U[G.base + i * G.stride])));
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const double qmax = double((1 << (bits - 1)) - 1), qmin = -qmax - 1.0;
    const double base = fmax(amax / qmax, 1e-8);
    if (lane == 0) scale_out[g] = base;
    if (!mse) return;
    for (int c0 = 0; c0 < kCands; c0 += 32) {
        const int cand = c0 + lane;
        const double s = grid_scale(base, cand < kCands ? cand : 0);
        double err = 0.0;
        for (long long i = 0; i < G.count; ++i)
            err = __dadd_rn(err, mse_term(double(U[G.base + i * G.stride]), s, qmax, qmin));
        if (cand < kCands) err_out[(long long)g * kCands + cand] = err;
    }
}

// scale_mse_grid's selection (quant.cpp:122-134): start from the MinMax scale, take a grid
// point only on a strict improvement, in grid order.
__global__ void k_pick_best(int groups, const double* __restrict__ err, double* __restrict__ scale) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= groups) return;
    const double base = scale[g];
    double best = base, best_err = err[(long long)g * kCands];
    for (int c = 1; c < kCands; ++c) {
        const double e = err[(long long)g * kCands + c];
        if (e < best_err) best_err = e, best = grid_scale(base, c);
    }
    scale[g] = best;
}

// uq[f][oc][ic] = quantize_value(U, fil(oc, f)) (quant.cpp:221-229) and the expanded table
// fil_full[oc * F + f] the fp64 output epilogue reads.  QT = int8_t (bits <= 8, the
// tensor-core operand) or double (bits 9-16: integer-valued fp64 for the exact fp64 GEMM).
template <class TU, class QT>
__global__ void k_fil_quantize(const TU* __restrict__ U, int OC, int IC, int F, int scope,
                               const double* __restrict__ scale, int bits, int Cpad, int OCpad,
                               QT* __restrict__ uqB, double* __restrict__ fil_full,
                               unsigned long long* __restrict__ sat) {
    const long long n = (long long)OC * IC * F;
    const int qmax = (1 << (bits - 1)) - 1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int f = int(i % F), ic = int((i / F) % IC), oc = int(i / ((long long)F * IC));
        const double s = scope == 0 ? scale[oc] : (scope == 1 ? scale[f] : scale[(long long)oc * F + f]);
        uqB[((long long)f * OCpad + oc) * Cpad + ic] = QT(clamp_q(int(rint(__ddiv_rn(double(U[i]), s))), qmax, sat));
        if (ic == 0) fil_full[(long long)oc * F + f] = s;
    }
}

// Per-frequency max|V| over the kept V [F][Tpad][Cpad] (t < T, c < C): vmaxf[f].
// (maxima as the bit patterns of non-negative doubles, which order like the values)
template <class TV>
__global__ void __launch_bounds__(256) k_act_fmax(const TV* __restrict__ V, ConvGeom g, int F, int per_freq,
                                                  unsigned long long* __restrict__ vmaxf) {
    const int f = blockIdx.y;
    const long long n = (long long)g.T * g.C;
    double m = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long t = i / g.C, c = i % g.C;
        m = fmax(m, fabs(double(V[((long long)f * g.Tpad + t) * g.Cpad + c])));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0)
        atomicMax(&vmaxf[per_freq ? f : 0], (unsigned long long)__double_as_longlong(m));
}

// MseGrid over this shard's V for every candidate of every activation group, continuing the
// reference's single sequential fp64 sum (quant.cpp:19-30) from err_in (the accumulators of
// the shards before this one in batch order; nullptr = the start of the batch): the batch
// split over ranks and chained rank by rank gives bitwise the full-batch sums.  Value order
// as quant.cpp:168-181: PerTensor = all of g.v in (tile, c, f) order, PerFrequency = (tile,
// c) for one f.  One block of 4 warps per group; lane = candidate (scales from the global
// maxima).
template <class TV>
__global__ void __launch_bounds__(128) k_act_mse(const TV* __restrict__ V, ConvGeom g, int F, int per_freq,
                                                 const unsigned long long* __restrict__ vmax, int bits,
                                                 const double* __restrict__ err_in, double* __restrict__ err_out) {
    const int grp = blockIdx.x, cand = threadIdx.x;
    if (cand >= kCands) return;
    const double qmax = double((1 << (bits - 1)) - 1), qmin = -qmax - 1.0;
    const double base = fmax(__longlong_as_double((long long)vmax[per_freq ? grp : 0]) / qmax, 1e-8);
    const double s = grid_scale(base, cand);
    double err = err_in ? err_in[grp * kCands + cand] : 0.0;
    const long long tc = (long long)g.T * g.C;
    if (per_freq) {
        const TV* Vf = V + (long long)grp * g.Tpad * g.Cpad;
        for (long long i = 0; i < tc; ++i) {
            const long long t = i / g.C, c = i - t * g.C;
            err = __dadd_rn(err, mse_term(double(Vf[t * g.Cpad + c]), s, qmax, qmin));
        }
    } else {
        for (long long i = 0; i < tc; ++i) {
            const long long t = i / g.C, c = i - t * g.C;
            for (int f = 0; f < F; ++f)
                err = __dadd_rn(err, mse_term(double(V[((long long)f * g.Tpad + t) * g.Cpad + c]), s, qmax, qmin));
        }
    }
    err_out[grp * kCands + cand] = err;
}

// Activation scales (quant.cpp:117-134): MinMax from the (global) maxima, or the MseGrid pick
// over the complete sums (the MinMax scale unless a grid point is strictly better, first wins).
__global__ void k_act_pick(int groups, int per_freq, const unsigned long long* __restrict__ vmax, int bits,
                           const double* __restrict__ err, double* __restrict__ act_scale) {
    const int grp = blockIdx.x * blockDim.x + threadIdx.x;
    if (grp >= groups) return;
    const double qmax = double((1 << (bits - 1)) - 1);
    const double base = fmax(__longlong_as_double((long long)vmax[per_freq ? grp : 0]) / qmax, 1e-8);
    if (!err) {
        act_scale[grp] = base;
        return;
    }
    double best = base, best_err = err[grp * kCands];
    for (int c = 1; c < kCands; ++c)
        if (err[grp * kCands + c] < best_err) best_err = err[grp * kCands + c], best = grid_scale(base, c);
    act_scale[grp] = best;
}

// vq[f][t][c] = quantize_value(V, sa(f)) (quant.cpp:242-250) for t < T, c < C (else 0);
// QT as in k_fil_quantize.
template <class TV, class QT>
__global__ void __launch_bounds__(256) k_quant_general(const TV* __restrict__ V, ConvGeom g, int F,
                                                       int per_freq, const double* __restrict__ act_scale, int bits,
                                                       QT* __restrict__ vqA, unsigned long long* __restrict__ sat) {
    const int f = blockIdx.y;
    const double s = act_scale[per_freq ? f : 0];
    const int qmax = (1 << (bits - 1)) - 1;
    const long long n = (long long)g.T * g.Cpad;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long t = i / g.Cpad, c = i - t * g.Cpad;
        const long long off = ((long long)f * g.Tpad + t) * g.Cpad + c;
        vqA[off] = c < g.C ? QT(clamp_q(int(rint(__ddiv_rn(double(V[off]), s))), qmax, sat)) : QT(0);
    }
}

// ---------------------------------------------------------------- real-valued inputs
// V = B^T x B for fp64 inputs in gather_tiles' exact order (quant.cpp:76-89): sequential
// sums over k, coefficients in {-1, 0, 1} (exact products, zero terms skipped: adding an
// exact zero leaves the value unchanged).  One thread per (tile, channel); V [F][Tpad][Cpad].
template <int V>
__global__ void __launch_bounds__(128) k_act_f64(const double* __restrict__ x, ConvGeom g, double* __restrict__ Vd) {
    using T = Tab<V>;
    constexpr int n = T::n, K = T::K, M = T::M;
    const long long item = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= (long long)g.T * g.C) return;
    const int c = int(item % g.C), t = int(item / g.C);
    const int tj = t % g.tw, ti = (t / g.tw) % g.th, b = t / (g.tw * g.th);
    const int ih0 = ti * M - g.pad, iw0 = tj * M - g.pad;
    const double* xc = x + ((size_t)b * g.C + c) * g.H * g.W;
    double win[n][n];
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int s2 = 0; s2 < n; ++s2) {
            const int ih = ih0 + r, iw = iw0 + s2;
            win[r][s2] = (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) ? xc[(size_t)ih * g.W + iw] : 0.0;
        }
    for (int i = 0; i < K; ++i) {
        double tmp[n];
#pragma unroll
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < n; ++k) {
                const int bt = T::bt(i, k);
                if (bt) acc = __dadd_rn(acc, bt > 0 ? win[k][j] : -win[k][j]);
            }
            tmp[j] = acc;
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < n; ++k) {
                const int bt = T::bt(j, k);
                if (bt) acc = __dadd_rn(acc, bt > 0 ? tmp[k] : -tmp[k]);
            }
            Vd[((size_t)(i * K + j) * g.Tpad + t) * g.Cpad + c] = acc;
        }
    }
}

// U = G f G^T for fp64 filters in transform_filters' order (conv.cpp:362-380); U [OC][IC][F].
template <int V>
__global__ void __launch_bounds__(128) k_filters_f64(const double* __restrict__ w, int OC, int IC,
                                                     double* __restrict__ U) {
    using T = Tab<V>;
    constexpr int R = T::R, K = T::K;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)OC * IC) return;
    const double* f = w + idx * R * R;
    double tmp[K][R];
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int gk = T::g(i, k);
                if (gk) acc = __dadd_rn(acc, gk > 0 ? f[k * R + j] : -f[k * R + j]);
            }
            tmp[i][j] = acc;
        }
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = 0; j < K; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int gk = T::g(j, k);
                if (gk) acc = __dadd_rn(acc, gk > 0 ? tmp[i][k] : -tmp[i][k]);
            }
            U[idx * T::F + i * K + j] = acc;
        }
}

// direct_conv2d (conv.cpp:320-350) in fp64, one output per thread, the reference's loop order.
__global__ void __launch_bounds__(256) k_direct_f64(const double* __restrict__ x, int B, int C, int H, int W,
                                                    const double* __restrict__ w, int OC, int R, int stride, int pad,
                                                    int HO, int WO, double* __restrict__ out) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)B * OC * HO * WO) return;
    const int ow = int(idx % WO), oh = int((idx / WO) % HO), oc = int((idx / ((long long)WO * HO)) % OC);
    const int b = int(idx / ((long long)WO * HO * OC));
    double acc = 0.0;
    for (int ic = 0; ic < C; ++ic)
        for (int fr = 0; fr < R; ++fr) {
            const int ih = oh * stride - pad + fr;
            if (ih < 0 || ih >= H) continue;
            for (int fc = 0; fc < R; ++fc) {
                const int iw = ow * stride - pad + fc;
                if (iw < 0 || iw >= W) continue;
                acc = __dadd_rn(acc, __dmul_rn(x[((size_t(b) * C + ic) * H + ih) * W + iw],
                                               w[((size_t(oc) * C + ic) * R + fr) * R + fc]));
            }
        }
    out[idx] = acc;
}

// U [OC][IC][F] -> the float path's GEMM operand Ub [F][OCpad][Cpad] (zero padding done by the caller).
__global__ void k_pack_u_f64(const double* __restrict__ U, int OC, int IC, int F, int Cpad, int OCpad,
                             double* __restrict__ Ub) {
    const long long n = (long long)OC * IC * F;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int f = int(i % F), ic = int((i / F) % IC), oc = int(i / ((long long)F * IC));
        Ub[((long long)f * OCpad + oc) * Cpad + ic] = U[i];
    }
}

// Reduced batch of the paired schedule: dst[s][e] = sum_k coef[k] * src[f_k][e], the
// evaluation form accumulated in the reference's order (conv.cpp:482-489).
__global__ void k_pair_gather(const double* __restrict__ src, long long elems, const PairSlice* __restrict__ tab,
                              bool filter_side, double* __restrict__ dst) {
    const PairSlice sl = tab[blockIdx.y];
    double* out = dst + (long long)blockIdx.y * elems;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < elems;
         e += (long long)gridDim.x * blockDim.x) {
        if (sl.n == 1) {
            out[e] = src[(long long)sl.f[0] * elems + e];
            continue;
        }
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            acc = __dadd_rn(acc, __dmul_rn(filter_side ? sl.b[k] : sl.a[k], src[(long long)sl.f[k] * elems + e]));
        out[e] = acc;
    }
}

// P[f][e] from the reduced batch: direct copy, zero, or a corner fold (conv.cpp:494-506).
__global__ void k_pair_fold(const double* __restrict__ Pr, long long elems, const PairFold* __restrict__ tab,
                            double* __restrict__ P) {
    const PairFold fd = tab[blockIdx.y];
    double* out = P + (long long)blockIdx.y * elems;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < elems;
         e += (long long)gridDim.x * blockDim.x) {
        double v = 0.0;
        if (fd.kind == 1) {
            v = Pr[(long long)fd.src * elems + e];
        } else if (fd.kind == 2) {
#pragma unroll
            for (int l = 0; l < 6; ++l) v = __dadd_rn(v, __dmul_rn(fd.w[l], Pr[(long long)(fd.src + l) * elems + e]));
        }
        out[e] = v;
    }
}

// ============================================================================ host
namespace {
template <class TU>
cudaError_t fil_general(const TU* U, int OC, int IC, int F, int scope, int mse, int bits, int Cpad, int OCpad,
                        double* scale_native, double* err_tmp, void* uqB, double* fil_full, unsigned long long* sat,
                        cudaStream_t st) {
    const int groups = scope == 0 ? OC : (scope == 1 ? F : OC * F);
    k_fil_scales<TU><<<groups, 32, 0, st>>>(U, OC, IC, F, scope, mse, bits, scale_native, err_tmp);
    if (mse) k_pick_best<<<(groups + 127) / 128, 128, 0, st>>>(groups, err_tmp, scale_native);
    const long long n = (long long)OC * IC * F;
    const int blocks = int((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    if (bits > 8)
        k_fil_quantize<TU, double><<<blocks, 256, 0, st>>>(U, OC, IC, F, scope, scale_native, bits, Cpad, OCpad,
                                                           static_cast<double*>(uqB), fil_full, sat);
    else
        k_fil_quantize<TU, int8_t><<<blocks, 256, 0, st>>>(U, OC, IC, F, scope, scale_native, bits, Cpad, OCpad,
                                                           static_cast<int8_t*>(uqB), fil_full, sat);
    return cudaGetLastError();
}

template <class TV>
cudaError_t act_maxima(const TV* V, const ConvGeom& g, int F, int per_freq, unsigned long long* vmax,
                       cudaStream_t st) {
    const long long n = (long long)g.T * g.C;
    const int bx = int((n + 255) / 256 < 64 ? (n + 255) / 256 : 64);
    k_act_fmax<TV><<<dim3(bx, F), 256, 0, st>>>(V, g, F, per_freq, vmax);
    return cudaGetLastError();
}

template <class TV>
cudaError_t act_mse(const TV* V, const ConvGeom& g, int F, int per_freq, const unsigned long long* vmax, int bits,
                    const double* err_in, double* err_out, cudaStream_t st) {
    k_act_mse<TV><<<per_freq ? F : 1, 128, 0, st>>>(V, g, F, per_freq, vmax, bits, err_in, err_out);
    return cudaGetLastError();
}

cudaError_t act_pick(int F, int per_freq, const unsigned long long* vmax, int bits, const double* err,
                     double* act_scale, cudaStream_t st) {
    const int groups = per_freq ? F : 1;
    k_act_pick<<<(groups + 127) / 128, 128, 0, st>>>(groups, per_freq, vmax, bits, err, act_scale);
    return cudaGetLastError();
}

template <class TV>
cudaError_t act_quantize(const TV* V, const ConvGeom& g, int F, int per_freq, const double* act_scale, int bits,
                         void* vqA, unsigned long long* sat, cudaStream_t st) {
    const long long nq = (long long)g.T * g.Cpad;
    const int bq = int((nq + 255) / 256 < 64 ? (nq + 255) / 256 : 64);
    if (bits > 8)
        k_quant_general<TV, double><<<dim3(bq, F), 256, 0, st>>>(V, g, F, per_freq, act_scale, bits,
                                                                 static_cast<double*>(vqA), sat);
    else
        k_quant_general<TV, int8_t><<<dim3(bq, F), 256, 0, st>>>(V, g, F, per_freq, act_scale, bits,
                                                                 static_cast<int8_t*>(vqA), sat);
    return cudaGetLastError();
}

template <class TV>
cudaError_t act_general(const TV* V, const ConvGeom& g, int F, int per_freq, int mse, int bits,
                        unsigned long long* vmax, double* act_scale, void* vqA, unsigned long long* sat,
                        double* err_tmp, cudaStream_t st) {
    cudaError_t e = act_maxima(V, g, F, per_freq, vmax, st);
    if (e == cudaSuccess && mse) e = act_mse(V, g, F, per_freq, vmax, bits, nullptr, err_tmp, st);
    if (e == cudaSuccess) e = act_pick(F, per_freq, vmax, bits, mse ? err_tmp : nullptr, act_scale, st);
    if (e == cudaSuccess) e = act_quantize(V, g, F, per_freq, act_scale, bits, vqA, sat, st);
    return e;
}
}  // namespace

cudaError_t launch_fil_general(const int32_t* U, int OC, int IC, int F, int scope, int mse, int bits, int Cpad,
                               int OCpad, double* scale_native, double* err_tmp, void* uqB, double* fil_full,
                               unsigned long long* sat, cudaStream_t st) {
    return fil_general(U, OC, IC, F, scope, mse, bits, Cpad, OCpad, scale_native, err_tmp, uqB, fil_full, sat, st);
}

cudaError_t launch_fil_general_f64(const double* U, int OC, int IC, int F, int scope, int mse, int bits, int Cpad,
                                   int OCpad, double* scale_native, double* err_tmp, void* uqB, double* fil_full,
                                   unsigned long long* sat, cudaStream_t st) {
    return fil_general(U, OC, IC, F, scope, mse, bits, Cpad, OCpad, scale_native, err_tmp, uqB, fil_full, sat, st);
}

cudaError_t launch_act_general(const int16_t* V, const ConvGeom& g, int F, int per_freq, int mse, int bits,
                               unsigned long long* vmax, double* act_scale, void* vqA, unsigned long long* sat,
                               double* err_tmp, cudaStream_t st) {
    return act_general(V, g, F, per_freq, mse, bits, vmax, act_scale, vqA, sat, err_tmp, st);
}

cudaError_t launch_act_general_f64(const double* V, const ConvGeom& g, int F, int per_freq, int mse, int bits,
                                   unsigned long long* vmax, double* act_scale, void* vqA, unsigned long long* sat,
                                   double* err_tmp, cudaStream_t st) {
    return act_general(V, g, F, per_freq, mse, bits, vmax, act_scale, vqA, sat, err_tmp, st);
}

cudaError_t launch_act_maxima(const int16_t* V, const ConvGeom& g, int F, int per_freq, unsigned long long* vmax,
                              cudaStream_t st) {
    return act_maxima(V, g, F, per_freq, vmax, st);
}

cudaError_t launch_act_mse(const int16_t* V, const ConvGeom& g, int F, int per_freq, const unsigned long long* vmax,
                           int bits, const double* err_in, double* err_out, cudaStream_t st) {
    return act_mse(V, g, F, per_freq, vmax, bits, err_in, err_out, st);
}

cudaError_t launch_act_pick(int F, int per_freq, const unsigned long long* vmax, int bits, const double* err,
                            double* act_scale, cudaStream_t st) {
    return act_pick(F, per_freq, vmax, bits, err, act_scale, st);
}

cudaError_t launch_act_quantize(const int16_t* V, const ConvGeom& g, int F, int per_freq, const double* act_scale,
                                int bits, void* vqA, unsigned long long* sat, cudaStream_t st) {
    return act_quantize(V, g, F, per_freq, act_scale, bits, vqA, sat, st);
}

cudaError_t launch_act_f64(int variant, const double* x, const ConvGeom& g, double* Vd, cudaStream_t st) {
    const long long n = (long long)g.T * g.C;
    const int blocks = int((n + 127) / 128);
    switch (variant) {
        case 0: k_act_f64<0><<<blocks, 128, 0, st>>>(x, g, Vd); break;
        case 1: k_act_f64<1><<<blocks, 128, 0, st>>>(x, g, Vd); break;
        case 2: k_act_f64<2><<<blocks, 128, 0, st>>>(x, g, Vd); break;
        case 3: k_act_f64<3><<<blocks, 128, 0, st>>>(x, g, Vd); break;
        default: k_act_f64<4><<<blocks, 128, 0, st>>>(x, g, Vd); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_filters_f64(int variant, const double* w, int OC, int IC, double* U, cudaStream_t st) {
    const long long n = (long long)OC * IC;
    const int blocks = int((n + 127) / 128);
    switch (variant) {
        case 0: k_filters_f64<0><<<blocks, 128, 0, st>>>(w, OC, IC, U); break;
        case 1: k_filters_f64<1><<<blocks, 128, 0, st>>>(w, OC, IC, U); break;
        case 2: k_filters_f64<2><<<blocks, 128, 0, st>>>(w, OC, IC, U); break;
        case 3: k_filters_f64<3><<<blocks, 128, 0, st>>>(w, OC, IC, U); break;
        default: k_filters_f64<4><<<blocks, 128, 0, st>>>(w, OC, IC, U); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_pack_u_f64(const double* U, int OC, int IC, int F, int Cpad, int OCpad, double* Ub,
                              cudaStream_t st) {
    const long long n = (long long)OC * IC * F;
    const int blocks = int((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    k_pack_u_f64<<<blocks, 256, 0, st>>>(U, OC, IC, F, Cpad, OCpad, Ub);
    return cudaGetLastError();
}

cudaError_t launch_pair_gather(const double* src, long long elems, const PairSlice* tab, int nslices, bool filter_side,
                               double* dst, cudaStream_t st) {
    const long long bx = (elems + 255) / 256;
    const dim3 grid(unsigned(bx < 64 ? bx : 64), unsigned(nslices));
    k_pair_gather<<<grid, 256, 0, st>>>(src, elems, tab, filter_side, dst);
    return cudaGetLastError();
}

cudaError_t launch_pair_fold(const double* Pr, long long elems, const PairFold* tab, int F, double* P,
                             cudaStream_t st) {
    const long long bx = (elems + 255) / 256;
    const dim3 grid(unsigned(bx < 64 ? bx : 64), unsigned(F));
    k_pair_fold<<<grid, 256, 0, st>>>(Pr, elems, tab, P);
    return cudaGetLastError();
}

cudaError_t launch_direct_f64(const double* x, int B, int C, int H, int W, const double* w, int OC, int R, int stride,
                              int pad, double* out, cudaStream_t st) {
    const int HO = (H + 2 * pad - R) / stride + 1, WO = (W + 2 * pad - R) / stride + 1;
    const long long n = (long long)B * OC * HO * WO;
    k_direct_f64<<<int((n + 255) / 256), 256, 0, st>>>(x, B, C, H, W, w, OC, R, stride, pad, HO, WO, out);
    return cudaGetLastError();
}

}  // namespace sfcb200
