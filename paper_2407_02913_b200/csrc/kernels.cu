// CUDA kernels for the quantized SFC 3x3 convolution on sm_100a.
//
// Pipeline (reference: proj/src/quant.cpp:152-293):
//   k_filter_prepare   U = G f G^T, per-oc minmax scale, exact RNE quantize   (conv.cpp:352-382, quant.cpp:183-229)
//   k_act_transform<0> V = BT x BT^T over every tile/channel, global max|V|   (quant.cpp:44-93, 168-172)
//   k_quant_params     sa and an exhaustively verified integer quantizer      (quant.cpp:102-120)
//   k_act_transform<1> V -> vq (int8) in the GEMM A-operand layout             (quant.cpp:242-250)
//   k_gemm             P_f = vq_f * uq_f^T on tcgen05 (kind::i8, TMEM int32)   (quant.cpp:251-257)
//   k_output           y = A^T P A (integer), dequantize / requantize          (quant.cpp:258-278)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <type_traits>

#include "ptx.cuh"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"

namespace sfcb200 {

namespace {
constexpr int kRowsPerTile = 128;  // GEMM M block (tiles per CTA)
constexpr int kChanPerCta = 32;    // channels per transform CTA

__device__ __forceinline__ int clamp_q(int q, int qmax, unsigned long long* sat) {
    const int qmin = -qmax - 1;
    if (q > qmax || q < qmin) {
        atomicAdd(sat, 1ull);
        q = q > qmax ? qmax : qmin;
    }
    return q;
}

// Exact activation quantizer: rint(double(v) / sa) clamped (quant.cpp:102-115).
__device__ __forceinline__ int quant_act(int v, const QuantParams& qp, unsigned long long* sat) {
    int q;
    if (qp.exact) {
        const long long p = (long long)v * qp.mul + (1ll << (qp.shift - 1));
        q = int(p >> qp.shift);
    } else {
        q = int(rint(__ddiv_rn(double(v), qp.sa)));
    }
    return clamp_q(q, qp.qmax, sat);
}
}  // namespace

// ============================================================================ filters
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
    auto transform = [&](int ic, int (&U)[T::K][T::K]) {
        int f[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) f[r][c] = w[((size_t(oc) * IC + ic) * 3 + r) * 3 + c];
#pragma unroll
        for (int k = 0; k < T::K; ++k) {
            int tmp[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                int acc = 0;
#pragma unroll
                for (int r = 0; r < 3; ++r) acc += T::g(k, r) * f[r][j];
                tmp[j] = acc;
            }
#pragma unroll
            for (int l = 0; l < T::K; ++l) {
                int acc = 0;
#pragma unroll
                for (int j = 0; j < 3; ++j) acc += tmp[j] * T::g(l, j);
                U[k][l] = acc;
            }
        }
    };
    for (int ic = threadIdx.x; ic < IC; ic += blockDim.x) {
        int U[T::K][T::K];
        transform(ic, U);
#pragma unroll
        for (int k = 0; k < T::K; ++k)
#pragma unroll
            for (int l = 0; l < T::K; ++l) local = max(local, abs(U[k][l]));
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
        int U[T::K][T::K];
        transform(ic, U);
#pragma unroll
        for (int k = 0; k < T::K; ++k)
#pragma unroll
            for (int l = 0; l < T::K; ++l) {
                const int q = clamp_q(int(rint(__ddiv_rn(double(U[k][l]), sf))), qmax, sat);
                uqB[(size_t(k * T::K + l) * OCpad + oc) * Cpad + ic] = int8_t(q);
            }
    }
}

// ============================================================================ activations
// One CTA per (image b, tile row ti, chunk of 32 channels): the n input rows of
// the tile row are staged in shared memory (coalesced along W, zero outside the
// image exactly like quant.cpp:66-75), then each thread transforms one
// (tile column, channel) window.  QUANT=0 computes the global max|V|,
// QUANT=1 writes vq[f][t][c] (the K-major A operand of the per-frequency GEMMs).
template <int V, int QUANT>
__global__ void __launch_bounds__(256) k_act_transform(const int8_t* __restrict__ x, ConvGeom g,
                                                       int* __restrict__ vmax, const QuantParams* __restrict__ qpp,
                                                       int8_t* __restrict__ vqA, unsigned long long* sat) {
    using T = Tab<V>;
    extern __shared__ int8_t s_in[];  // [kChanPerCta][n][wcols]
    const int ti = blockIdx.x, b = blockIdx.y, c0 = blockIdx.z * kChanPerCta;
    const int nch = min(kChanPerCta, g.C - c0);
    const int wcols = (g.tw - 1) * T::M + T::n;
    const int ih0 = ti * T::M - g.pad, iw0 = -g.pad;
    for (int i = threadIdx.x; i < nch * T::n * wcols; i += blockDim.x) {
        const int col = i % wcols, r = (i / wcols) % T::n, c = i / (wcols * T::n);
        const int ih = ih0 + r, iw = iw0 + col;
        int8_t v = 0;
        if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) v = x[((size_t(b) * g.C + c0 + c) * g.H + ih) * g.W + iw];
        s_in[i] = v;
    }
    __syncthreads();
    QuantParams qp;
    if (QUANT) qp = *qpp;
    int local = 0;
    for (int item = threadIdx.x; item < nch * g.tw; item += blockDim.x) {
        const int c = item % nch, tj = item / nch;
        const int8_t* win = s_in + size_t(c) * T::n * wcols + tj * T::M;
        int xw[T::n][T::n];
#pragma unroll
        for (int r = 0; r < T::n; ++r)
#pragma unroll
            for (int s = 0; s < T::n; ++s) xw[r][s] = win[r * wcols + s];
        const int t = (b * g.th + ti) * g.tw + tj;
#pragma unroll
        for (int k = 0; k < T::K; ++k) {
            int row[T::n];  // (BT x)[k][:]
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
                if (QUANT) {
                    const int q = quant_act(v, qp, sat);
                    vqA[(size_t(k * T::K + l) * g.Tpad + t) * g.Cpad + c0 + c] = int8_t(q);
                } else {
                    local = max(local, abs(v));
                }
            }
        }
    }
    if (!QUANT) {
#pragma unroll
        for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
        if ((threadIdx.x & 31) == 0 && local > 0) atomicMax(vmax, local);
    }
}

// ============================================================================ scale
// sa = max(vmax / qmax, 1e-8) and a multiply-shift quantizer that reproduces
// rint(double(v) / sa) for every integer |v| <= vmax, verified exhaustively
// here (falls back to per-element fp64 division if no candidate is exact,
// e.g. when exact ties alternate their rounding direction).
__global__ void __launch_bounds__(1024) k_quant_params(const int* __restrict__ vmax_p, int bits,
                                                       QuantParams* __restrict__ qp, unsigned long long* sat) {
    const int vmax = *vmax_p;
    const int qmax = (1 << (bits - 1)) - 1;
    const double sa = fmax(double(vmax) / double(qmax), 1e-8);
    int e;
    frexp(sa, &e);
    const int shift = 29 + e;
    const long long m0 = (long long)floor(ldexp(1.0, shift) / sa);
    __shared__ int s_found;
    if (threadIdx.x == 0) s_found = -1;
    __syncthreads();
    for (int cand = 0; cand < 5; ++cand) {
        const long long mul = m0 + (cand == 0 ? 0 : (cand & 1 ? (cand + 1) / 2 : -(cand / 2)));
        int bad = 0;
        for (int v = -vmax + int(threadIdx.x); v <= vmax; v += blockDim.x) {
            const long long fast = ((long long)v * mul + (1ll << (shift - 1))) >> shift;
            const long long ref = (long long)rint(__ddiv_rn(double(v), sa));
            bad |= fast != ref;
        }
        bad = __syncthreads_or(bad);
        if (!bad) {
            if (threadIdx.x == 0) s_found = cand;
            break;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *sat = 0;  // activation saturation counter of this call
        QuantParams p;
        p.sa = sa;
        p.shift = shift;
        p.vmax = vmax;
        p.qmax = qmax;
        p.exact = s_found >= 0;
        const int cand = s_found >= 0 ? s_found : 0;
        p.mul = m0 + (cand == 0 ? 0 : (cand & 1 ? (cand + 1) / 2 : -(cand / 2)));
        *qp = p;
    }
}

// ============================================================================ GEMM
// P[f][t][oc] = sum_ic vq[f][t][ic] * uq[f][oc][ic] for the frequencies
// f0 .. f0+nf-1 of this CTA.  Warp-specialized: warp 0 = TMA producer,
// warp 1 = tcgen05 issuer (+ TMEM owner), warps 2-5 = epilogue (TMEM -> HBM).
// Accumulators are double-buffered in TMEM across frequencies.
template <int BN, int BK, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int32_t* __restrict__ P,
           int Tpad, int OCpad, int Cpad, int F, int fgroup) {
    constexpr int kTmemCols = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
    constexpr uint32_t kStageBytes = (kRowsPerTile + BN) * BK;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = sA + STAGES * kRowsPerTile * BK;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * BN * BK);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tb = blockIdx.x, ob = blockIdx.y, f0 = blockIdx.z * fgroup;
    const int nf = min(fgroup, F - f0);
    const int nk = Cpad / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tmem_holder, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {
            ptx::tma_prefetch(&tmA);
            ptx::tma_prefetch(&tmB);
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0; i < nf; ++i)
                for (int kc = 0; kc < nk; ++kc) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_expect_tx(&full[stage], kStageBytes);
                    ptx::tma_load_3d(sA + stage * kRowsPerTile * BK, &tmA, &full[stage], kc * BK, tb * kRowsPerTile,
                                     f0 + i);
                    ptx::tma_load_3d(sB + stage * BN * BK, &tmB, &full[stage], kc * BK, ob * BN, f0 + i);
                    if (++stage == STAGES) stage = 0, phase ^= 1;
                }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_i8(kRowsPerTile, BN);
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0; i < nf; ++i) {
                const int ab = i & 1;
                const uint32_t use = uint32_t(i >> 1);
                ptx::mbar_wait(&tempty[ab], (use & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + uint32_t(ab * BN);
                for (int kc = 0; kc < nk; ++kc) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(sA + stage * kRowsPerTile * BK);
                    const uint32_t b0 = ptx::smem_u32(sB + stage * BN * BK);
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk)
                        ptx::mma_i8(d, ptx::smem_desc_kmajor(a0 + kk * 32, BK), ptx::smem_desc_kmajor(b0 + kk * 32, BK),
                                    idesc, (kc | kk) != 0);
                    ptx::mma_commit(&empty[stage]);
                    if (++stage == STAGES) stage = 0, phase ^= 1;
                }
                ptx::mma_commit(&tfull[ab]);
            }
        }
    } else {
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int row = tb * kRowsPerTile + q * 32 + lane;
        for (int i = 0; i < nf; ++i) {
            const int ab = i & 1;
            const uint32_t use = uint32_t(i >> 1);
            ptx::mbar_wait(&tfull[ab], use & 1);
            ptx::tc_fence_after();
            int32_t* dst = P + (size_t(f0 + i) * Tpad + row) * OCpad + size_t(ob) * BN;
#pragma unroll 1
            for (int c = 0; c < BN; c += 16) {
                int32_t r[16];
                ptx::tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(ab * BN + c), r);
                ptx::tmem_wait_ld();
                int4* d4 = reinterpret_cast<int4*>(dst + c);
                d4[0] = make_int4(r[0], r[1], r[2], r[3]);
                d4[1] = make_int4(r[4], r[5], r[6], r[7]);
                d4[2] = make_int4(r[8], r[9], r[10], r[11]);
                d4[3] = make_int4(r[12], r[13], r[14], r[15]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[ab]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, kTmemCols);
    }
}

// ============================================================================ output
// One thread per (tile, oc): y[t1][t2] = sum_l (sum_k A[k,t1] P[k,l]) A[l,t2]
// in exact integers, then fp32 out = y * sa * sf[oc] / N^2 and / or the
// harness int8 requant clamp(rint(out * s), 0, 127).
template <int V, bool Y64>
__global__ void __launch_bounds__(128) k_output(const int32_t* __restrict__ P, ConvGeom g,
                                                const QuantParams* __restrict__ qpp, const double* __restrict__ sf,
                                                double requant, int32_t* __restrict__ y32, int64_t* __restrict__ y64,
                                                float* __restrict__ out, int8_t* __restrict__ out8) {
    using T = Tab<V>;
    using acc_t = typename std::conditional<Y64, long long, int>::type;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)g.T * g.OC) return;
    const int oc = int(idx % g.OC), t = int(idx / g.OC);
    const int per_img = g.th * g.tw;
    const int b = t / per_img, ti = (t % per_img) / g.tw, tj = t % g.tw;
    acc_t y[T::M][T::M];
#pragma unroll
    for (int i = 0; i < T::M; ++i)
#pragma unroll
        for (int j = 0; j < T::M; ++j) y[i][j] = 0;
#pragma unroll
    for (int l = 0; l < T::K; ++l) {
        int p[T::K];
#pragma unroll
        for (int k = 0; k < T::K; ++k) p[k] = P[(size_t(k * T::K + l) * g.Tpad + t) * g.OCpad + oc];
#pragma unroll
        for (int t1 = 0; t1 < T::M; ++t1) {
            int qv = 0;
#pragma unroll
            for (int k = 0; k < T::K; ++k)
                if (T::a(k, t1) != 0) qv += T::a(k, t1) * p[k];
#pragma unroll
            for (int t2 = 0; t2 < T::M; ++t2)
                if (T::a(l, t2) != 0) y[t1][t2] += acc_t(qv) * T::a(l, t2);
        }
    }
    const double scale = (qpp->sa * sf[oc]) / double(T::DEN * T::DEN);
#pragma unroll
    for (int t1 = 0; t1 < T::M; ++t1) {
        const int oh = ti * T::M + t1;
        if (oh >= g.HO) break;
#pragma unroll
        for (int t2 = 0; t2 < T::M; ++t2) {
            const int ow = tj * T::M + t2;
            if (ow >= g.WO) break;
            const size_t o = ((size_t(b) * g.OC + oc) * g.HO + oh) * g.WO + ow;
            if (y32) y32[o] = int(y[t1][t2]);
            if (y64) y64[o] = (long long)y[t1][t2];
            const double val = double(y[t1][t2]) * scale;
            if (out) out[o] = float(val);
            if (out8) out8[o] = int8_t(fmin(fmax(rint(val * requant), 0.0), 127.0));
        }
    }
}

// ============================================================================ host side
namespace {
int variant_M(int v) { return v == 0 ? Tab<0>::M : v == 1 ? Tab<1>::M : Tab<2>::M; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool make_tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                  uint32_t b1) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0, d0 * d1};
    cuuint32_t box[3] = {b0, b1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUtensorMapSwizzle sw = b0 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : b0 == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int BN, int BK>
cudaError_t gemm_launch(const CUtensorMap& a, const CUtensorMap& b, int32_t* P, const ConvGeom& g, int F,
                        cudaStream_t st) {
    constexpr int STAGES = 4;
    const size_t smem = size_t(STAGES) * (kRowsPerTile + BN) * BK + 1024 + 256;
    auto kern = k_gemm<BN, BK, STAGES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const int tblocks = g.Tpad / kRowsPerTile, oblocks = g.OCpad / BN;
    // Enough frequency groups for about two waves over the 148 SMs.
    int groups = (2 * 148 + tblocks * oblocks - 1) / (tblocks * oblocks);
    groups = groups < 1 ? 1 : (groups > F ? F : groups);
    const int fgroup = (F + groups - 1) / groups;
    groups = (F + fgroup - 1) / fgroup;
    dim3 grid(tblocks, oblocks, groups);
    kern<<<grid, 192, smem, st>>>(a, b, P, g.Tpad, g.OCpad, g.Cpad, F, fgroup);
    return cudaGetLastError();
}
}  // namespace

void geom_init(ConvGeom& g, int variant, int B, int C, int H, int W, int pad, int OC) {
    const int M = variant_M(variant);
    g.B = B, g.C = C, g.H = H, g.W = W, g.pad = pad, g.OC = OC;
    g.HO = H + 2 * pad - 2;
    g.WO = W + 2 * pad - 2;
    g.th = (g.HO + M - 1) / M;
    g.tw = (g.WO + M - 1) / M;
    g.T = B * g.th * g.tw;
    g.Tpad = (g.T + kRowsPerTile - 1) / kRowsPerTile * kRowsPerTile;
    g.BK = C > 64 ? 128 : 64;
    g.Cpad = (C + g.BK - 1) / g.BK * g.BK;
    g.BN = OC <= 64 ? 64 : (OC <= 128 ? 128 : 256);
    g.OCpad = (OC + g.BN - 1) / g.BN * g.BN;
}

size_t workspace_bytes(const ConvGeom& g, int F) {
    auto up = [](size_t v) { return (v + 255) / 256 * 256; };
    return up(256) + up(size_t(F) * g.Tpad * g.Cpad) + up(size_t(F) * g.Tpad * g.OCpad * 4);
}

cudaError_t launch_filter_prepare(int variant, const int8_t* w, int OC, int IC, int Cpad, int OCpad, int bits,
                                  double* sf, int* umax, int8_t* uqB, unsigned long long* sat, cudaStream_t st) {
    switch (variant) {
        case 0: k_filter_prepare<0><<<OC, 128, 0, st>>>(w, OC, IC, Cpad, OCpad, bits, sf, umax, uqB, sat); break;
        case 1: k_filter_prepare<1><<<OC, 128, 0, st>>>(w, OC, IC, Cpad, OCpad, bits, sf, umax, uqB, sat); break;
        default: k_filter_prepare<2><<<OC, 128, 0, st>>>(w, OC, IC, Cpad, OCpad, bits, sf, umax, uqB, sat); break;
    }
    return cudaGetLastError();
}

template <int V, int Q>
static cudaError_t act_launch(const int8_t* x, const ConvGeom& g, int* vmax, const QuantParams* qp, int8_t* vqA,
                              unsigned long long* sat, cudaStream_t st) {
    const int wcols = (g.tw - 1) * Tab<V>::M + Tab<V>::n;
    const size_t smem = size_t(kChanPerCta) * Tab<V>::n * wcols;
    auto kern = k_act_transform<V, Q>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    dim3 grid(g.th, g.B, (g.C + kChanPerCta - 1) / kChanPerCta);
    kern<<<grid, 256, smem, st>>>(x, g, vmax, qp, vqA, sat);
    return cudaGetLastError();
}

cudaError_t launch_act_absmax(int variant, const int8_t* x, const ConvGeom& g, int* vmax, cudaStream_t st) {
    switch (variant) {
        case 0: return act_launch<0, 0>(x, g, vmax, nullptr, nullptr, nullptr, st);
        case 1: return act_launch<1, 0>(x, g, vmax, nullptr, nullptr, nullptr, st);
        default: return act_launch<2, 0>(x, g, vmax, nullptr, nullptr, nullptr, st);
    }
}

cudaError_t launch_quant_params(const int* vmax, int bits, QuantParams* qp, unsigned long long* sat,
                                cudaStream_t st) {
    k_quant_params<<<1, 1024, 0, st>>>(vmax, bits, qp, sat);
    return cudaGetLastError();
}

cudaError_t launch_act_quant(int variant, const int8_t* x, const ConvGeom& g, const QuantParams* qp, int bits,
                             int8_t* vqA, unsigned long long* sat, cudaStream_t st) {
    (void)bits;
    switch (variant) {
        case 0: return act_launch<0, 1>(x, g, nullptr, qp, vqA, sat, st);
        case 1: return act_launch<1, 1>(x, g, nullptr, qp, vqA, sat, st);
        default: return act_launch<2, 1>(x, g, nullptr, qp, vqA, sat, st);
    }
}

cudaError_t launch_gemm(const int8_t* vqA, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F,
                        cudaStream_t st) {
    CUtensorMap ta, tb;
    if (!make_tmap_3d(&ta, vqA, g.Cpad, g.Tpad, F, g.BK, kRowsPerTile) ||
        !make_tmap_3d(&tb, uqB, g.Cpad, g.OCpad, F, g.BK, g.BN))
        return cudaErrorInvalidValue;
    if (g.BK == 128) {
        if (g.BN == 64) return gemm_launch<64, 128>(ta, tb, P, g, F, st);
        if (g.BN == 128) return gemm_launch<128, 128>(ta, tb, P, g, F, st);
        return gemm_launch<256, 128>(ta, tb, P, g, F, st);
    }
    if (g.BN == 64) return gemm_launch<64, 64>(ta, tb, P, g, F, st);
    if (g.BN == 128) return gemm_launch<128, 64>(ta, tb, P, g, F, st);
    return gemm_launch<256, 64>(ta, tb, P, g, F, st);
}

template <int V>
static cudaError_t output_launch(bool y64, const int32_t* P, const ConvGeom& g, const QuantParams* qp,
                                 const double* sf, double requant, int32_t* y32, int64_t* y64p, float* out,
                                 int8_t* out8, cudaStream_t st) {
    const long long n = (long long)g.T * g.OC;
    const int blocks = int((n + 127) / 128);
    if (y64)
        k_output<V, true><<<blocks, 128, 0, st>>>(P, g, qp, sf, requant, y32, y64p, out, out8);
    else
        k_output<V, false><<<blocks, 128, 0, st>>>(P, g, qp, sf, requant, y32, y64p, out, out8);
    return cudaGetLastError();
}

cudaError_t launch_output(int variant, bool y64, const int32_t* P, const ConvGeom& g, const QuantParams* qp,
                          const double* sf, double requant, int32_t* y32, int64_t* y64p, float* out, int8_t* out8,
                          cudaStream_t st) {
    switch (variant) {
        case 0: return output_launch<0>(y64, P, g, qp, sf, requant, y32, y64p, out, out8, st);
        case 1: return output_launch<1>(y64, P, g, qp, sf, requant, y32, y64p, out, out8, st);
        default: return output_launch<2>(y64, P, g, qp, sf, requant, y32, y64p, out, out8, st);
    }
}

// ============================================================================ auxiliary (report / API) kernels
// Exact int8 correlation with int32 accumulation (direct_conv2d, conv.cpp:320-350).
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
                acc += int(x[((size_t(b) * C + ic) * H + ih) * W + iw]) * int(w[((size_t(oc) * C + ic) * R + fr) * R + fc]);
            }
        }
    out[idx] = acc;
}

// sum over tiles and channels of V[k][l]^2, exact in uint64 (frequency_energy, quant.cpp:136-150).
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
                xw[r][s] = (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) ? int(x[((size_t(b) * g.C + c) * g.H + ih) * g.W + iw]) : 0;
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

// U = G f G^T as exact int32 [OC][IC][K][K] (transform_filters, conv.cpp:352-382).
template <int V>
__global__ void __launch_bounds__(128) k_transform_filters(const int8_t* __restrict__ w, int OC, int IC,
                                                           int32_t* __restrict__ u) {
    using T = Tab<V>;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)OC * IC) return;
    int f[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) f[r][c] = w[idx * 9 + r * 3 + c];
#pragma unroll
    for (int k = 0; k < T::K; ++k) {
        int tmp[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            int acc = 0;
#pragma unroll
            for (int r = 0; r < 3; ++r) acc += T::g(k, r) * f[r][j];
            tmp[j] = acc;
        }
#pragma unroll
        for (int l = 0; l < T::K; ++l) {
            int acc = 0;
#pragma unroll
            for (int j = 0; j < 3; ++j) acc += tmp[j] * T::g(l, j);
            u[idx * T::F + k * T::K + l] = acc;
        }
    }
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
        default: k_freq_energy<2><<<blocks, 256, 0, st>>>(x, g, sum); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_transform_filters(int variant, const int8_t* w, int OC, int IC, int32_t* u, cudaStream_t st) {
    const long long n = (long long)OC * IC;
    const int blocks = int((n + 127) / 128);
    switch (variant) {
        case 0: k_transform_filters<0><<<blocks, 128, 0, st>>>(w, OC, IC, u); break;
        case 1: k_transform_filters<1><<<blocks, 128, 0, st>>>(w, OC, IC, u); break;
        default: k_transform_filters<2><<<blocks, 128, 0, st>>>(w, OC, IC, u); break;
    }
    return cudaGetLastError();
}

}  // namespace sfcb200

namespace sfcb200 {
// Debug / test hook: q(v) for every integer v in [-vmax, vmax] through the same device
// quantizer the activation kernel uses (fast multiply-shift or the fp64 fallback).
__global__ void k_debug_quant(const QuantParams* __restrict__ qpp, int vmax, int32_t* __restrict__ q,
                              unsigned long long* sat) {
    const QuantParams qp = *qpp;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= 2 * vmax; i += gridDim.x * blockDim.x)
        q[i] = quant_act(i - vmax, qp, sat);
}

cudaError_t launch_debug_quant(const QuantParams* qp, int vmax, int32_t* q, unsigned long long* sat, cudaStream_t st) {
    k_debug_quant<<<64, 256, 0, st>>>(qp, vmax, q, sat);
    return cudaGetLastError();
}
}  // namespace sfcb200
