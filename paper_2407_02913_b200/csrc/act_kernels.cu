// Activation stage of the quantized SFC conv: V = B^T x B per (tile, channel),
// the global max|V| pre-pass, and exact quantization into the GEMM A operand.
// Reference: gather_tiles (proj/src/quant.cpp:44-93), the PerTensor activation
// scale (quant.cpp:168-172) and the activation quantize loop (quant.cpp:242-250).
//
// One CTA per (image b, tile row ti, chunk of CC channels) covers every tile
// column of that tile row.  Thread t owns channel c = t % CC and work-group
// j = t / CC.  The transform is separable and runs in shared-memory stages:
//   stage 0  n input rows x wc columns, zero outside the image (quant.cpp:66-75)
//   stage 1  Z[tj][r][l] = sum_s BT[l][s] x[r][tj*M + s]      items (tj, r)
//   stage 2  V[k][l]     = sum_r BT[k][r] Z[tj][r][l]         items (tj, l)
//   stage 3  vq rows (f, t) <- shared staging, CC bytes each
// Every shared array is channel-innermost so a warp touches consecutive bytes,
// and all item decompositions divide by compile-time constants.
#include <cuda_runtime.h>

#include "common.cuh"
#include "ptx.cuh"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"
#include "transforms.cuh"

namespace sfcb200 {

namespace {
constexpr int kActThreads = 256;

struct ActSmem {
    int wcp;      // staged window columns per row, padded to 4
    int chs;      // bytes per staged channel (n * wcp, padded so chs / 4 is odd: conflict-free)
    size_t x_off, z_off, q_off, bytes;
};

template <int V, int CC>
__host__ __device__ inline ActSmem act_smem(int tw) {
    using T = Tab<V>;
    ActSmem s;
    s.wcp = ((tw - 1) * T::M + T::n + 3) & ~3;
    s.chs = T::n * s.wcp;
    if (((s.chs / 4) & 1) == 0) s.chs += 4;
    s.x_off = 0;
    s.z_off = (size_t(s.chs) * CC + 15) & ~size_t(15);
    s.q_off = s.z_off + ((size_t(tw) * T::n * T::K * CC * 2 + 15) & ~size_t(15));
    s.bytes = s.q_off + size_t(tw) * T::F * CC;
    return s;
}
}  // namespace

// MODE 0: max|V| -> atomicMax(*vmax).  MODE 1: quantize with the scale derived
// from *vmax_in and write vq[f][t][c] (row pitch Cpad) for f = k*K + l.
template <int V, int MODE, int CC>
__global__ void __launch_bounds__(kActThreads) k_act(const int8_t* __restrict__ x, ConvGeom g,
                                                     int* __restrict__ vmax, const int* __restrict__ vmax_in, int bits,
                                                     QuantParams* __restrict__ qp_out, int8_t* __restrict__ vqA,
                                                     unsigned long long* __restrict__ sat) {
    using T = Tab<V>;
    constexpr int n = T::n, K = T::K, M = T::M, F = T::F;
    constexpr int TPC = kActThreads / CC;   // work-groups per channel
    extern __shared__ __align__(16) uint8_t smem[];
    if (MODE == 0) griddep_launch_dependents();

    const int tw = g.tw;
    const int ti = blockIdx.x, b = blockIdx.y, c0 = blockIdx.z * CC;
    const int nch = min(CC, g.C - c0);
    const ActSmem L = act_smem<V, CC>(tw);
    int8_t* s_x = reinterpret_cast<int8_t*>(smem + L.x_off);     // [CC][n][wcp], channel stride chs
    int16_t* s_z = reinterpret_cast<int16_t*>(smem + L.z_off);   // [tw][n][K][CC]
    int8_t* s_q = reinterpret_cast<int8_t*>(smem + L.q_off);     // [tw][F][CC]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = threadIdx.x % CC, j = threadIdx.x / CC;

    // ---- stage 0: zero the staging area, then each warp copies whole channel segments:
    // the window rows [ih0, ih0 + n) of one channel are contiguous in NCHW, so lanes walk
    // that byte range coalesced and scatter into [c][r][pad + col] (32-bit index math).
    {
        uint4* z4 = reinterpret_cast<uint4*>(s_x);
        for (int i = threadIdx.x; i < (L.chs * CC) / 16; i += kActThreads) z4[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        const int ih0 = ti * M - g.pad;
        const int r_lo = max(ih0, 0), r_hi = min(ih0 + n, g.H);
        const int seg = (r_hi - r_lo) * g.W;                      // bytes per channel
        const unsigned wmagic = 0xffffffffu / unsigned(g.W) + 1;  // i / W == umulhi(i, wmagic) for i < 2^16
        const int8_t* src0 = x + (size_t(b) * g.C + c0) * size_t(g.H) * g.W + size_t(r_lo) * g.W;
        const int dst_row0 = (r_lo - ih0) * L.wcp + g.pad;
        for (int ch = warp; ch < nch; ch += kActThreads / 32) {
            const int8_t* src = src0 + size_t(ch) * g.H * g.W;
            int8_t* dst = s_x + ch * L.chs + dst_row0;
            for (int i = lane; i < seg; i += 32) {
                const int r = g.W == 1 ? i : int(__umulhi(unsigned(i), wmagic));
                dst[r * L.wcp + (i - r * g.W)] = src[i];
            }
        }
    }
    __syncthreads();

    // ---- stage 1: row transform, items (tj, r)
    for (int idx = j; idx < tw * n; idx += TPC) {
        const int r = idx % n, tj = idx / n;
        const int8_t* src = s_x + c * L.chs + r * L.wcp + tj * M;
        int xs[n];
#pragma unroll
        for (int s = 0; s < n; ++s) xs[s] = src[s];
        int16_t* dst = s_z + ((tj * n + r) * K) * CC + c;
        int z[K];
        fwd1d<V>(xs, z);
#pragma unroll
        for (int l = 0; l < K; ++l) dst[l * CC] = int16_t(z[l]);
    }

    QuantParams qp{};
    if (MODE == 1) {
        griddep_wait();  // the absmax pre-pass (and any multi-GPU MAX exchange) is complete
        qp = derive_qparams_block(*vmax_in, bits);  // contains __syncthreads
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) *qp_out = qp;
    } else {
        __syncthreads();
    }

    // ---- stage 2: column transform (+ quantize), items (tj, l)
    int local = 0;
    auto column = [&](auto quantize) {
        for (int idx = j; idx < tw * K; idx += TPC) {
            const int l = idx % K, tj = idx / K;
            int zr[n];
#pragma unroll
            for (int r = 0; r < n; ++r) zr[r] = s_z[((tj * n + r) * K + l) * CC + c];
            int v[K];
            fwd1d<V>(zr, v);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (MODE == 1)
                    s_q[(tj * F + k * K + l) * CC + c] = int8_t(quantize(v[k]));
                else
                    local = max(local, abs(v[k]));
            }
        }
    };
    if (MODE == 0) {
        column([](int v) { return v; });
    } else if (qp.exact) {  // uniform over the CTA: no per-value branch
        const long long mul = qp.mul, half = 1ll << (qp.shift - 1);
        const int shift = qp.shift;
        column([=](int v) { return int(((long long)v * mul + half) >> shift); });
    } else {
        column([&](int v) { return clamp_q(exact_q(v, qp.sa), qp.qmax, sat); });
    }

    if (MODE == 0) {
#pragma unroll
        for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
        if (lane == 0 && local > 0) atomicMax(vmax, local);
        return;
    }
    __syncthreads();
    griddep_launch_dependents();

    // ---- stage 3: CC contiguous bytes per vq row (f, t); channels >= C carry zeros
    constexpr int WPR = CC / 4;  // 32-bit words per row
    const int t0 = (b * g.th + ti) * tw;
    for (int i = threadIdx.x; i < tw * F * WPR; i += kActThreads) {
        const int wd = i % WPR, row = i / WPR;
        const int f = row % F, tj = row / F;
        const uint32_t v = reinterpret_cast<const uint32_t*>(s_q + size_t(row) * CC)[wd];
        reinterpret_cast<uint32_t*>(vqA + (size_t(f) * g.Tpad + t0 + tj) * g.Cpad + c0)[wd] = v;
    }
}

// Stand-alone quantizer derivation (stats / the exhaustive test hook).
__global__ void k_quant_params(const int* __restrict__ vmax_p, int bits, QuantParams* __restrict__ qp,
                               unsigned long long* sat) {
    const QuantParams p = derive_qparams_block(*vmax_p, bits);
    if (threadIdx.x == 0) {
        *qp = p;
        *sat = 0;
    }
}

__global__ void k_debug_quant(const QuantParams* __restrict__ qpp, int vmax, int32_t* __restrict__ q,
                              unsigned long long* sat) {
    const QuantParams qp = *qpp;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= 2 * vmax; i += gridDim.x * blockDim.x)
        q[i] = quant_act(i - vmax, qp, sat);
}

// ============================================================================ host
namespace {

template <int V, int MODE, int CC>
cudaError_t act_launch_cc(const int8_t* x, const ConvGeom& g, int* vmax, const int* vmax_in, int bits,
                          QuantParams* qp, int8_t* vqA, unsigned long long* sat, cudaStream_t st, bool pdl) {
    const size_t smem = act_smem<V, CC>(g.tw).bytes;
    auto kern = k_act<V, MODE, CC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.th, g.B, (g.C + CC - 1) / CC);
    cfg.blockDim = dim3(kActThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, x, g, vmax, vmax_in, bits, qp, vqA, sat);
}

// Channels per CTA: 32 gives full 32-byte vq row segments; shrink for two waves
// over the 148 SMs and a <= 96 KB shared-memory footprint.
template <int V>
int pick_cc(const ConvGeom& g) {
    auto ctas = [&](int c) { return long(g.th) * g.B * ((g.C + c - 1) / c); };
    auto smem = [&](int c) {
        return c == 32 ? act_smem<V, 32>(g.tw).bytes
             : c == 16 ? act_smem<V, 16>(g.tw).bytes
             : c == 8  ? act_smem<V, 8>(g.tw).bytes
                       : act_smem<V, 4>(g.tw).bytes;
    };
    int cc = 32;
    while (cc > 4 && ctas(cc) < 2 * 148) cc /= 2;
    while (cc > 4 && smem(cc) > 96 * 1024) cc /= 2;
    return cc;
}

template <int V, int MODE>
cudaError_t act_launch(const int8_t* x, const ConvGeom& g, int* vmax, const int* vmax_in, int bits, QuantParams* qp,
                       int8_t* vqA, unsigned long long* sat, cudaStream_t st, bool pdl) {
    switch (pick_cc<V>(g)) {
        case 32: return act_launch_cc<V, MODE, 32>(x, g, vmax, vmax_in, bits, qp, vqA, sat, st, pdl);
        case 16: return act_launch_cc<V, MODE, 16>(x, g, vmax, vmax_in, bits, qp, vqA, sat, st, pdl);
        case 8: return act_launch_cc<V, MODE, 8>(x, g, vmax, vmax_in, bits, qp, vqA, sat, st, pdl);
        default: return act_launch_cc<V, MODE, 4>(x, g, vmax, vmax_in, bits, qp, vqA, sat, st, pdl);
    }
}

}  // namespace

cudaError_t launch_act_absmax(int variant, const int8_t* x, const ConvGeom& g, int* vmax, cudaStream_t st) {
    switch (variant) {
        case 0: return act_launch<0, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, st, false);
        case 1: return act_launch<1, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, st, false);
        default: return act_launch<2, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, st, false);
    }
}

cudaError_t launch_act_quant(int variant, const int8_t* x, const ConvGeom& g, const int* vmax, int bits,
                             QuantParams* qp, int8_t* vqA, unsigned long long* sat, cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return act_launch<0, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, st, pdl);
        case 1: return act_launch<1, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, st, pdl);
        default: return act_launch<2, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, st, pdl);
    }
}

cudaError_t launch_quant_params(const int* vmax, int bits, QuantParams* qp, unsigned long long* sat,
                                cudaStream_t st) {
    k_quant_params<<<1, 256, 0, st>>>(vmax, bits, qp, sat);
    return cudaGetLastError();
}

cudaError_t launch_debug_quant(const QuantParams* qp, int vmax, int32_t* q, unsigned long long* sat,
                               cudaStream_t st) {
    k_debug_quant<<<64, 256, 0, st>>>(qp, vmax, q, sat);
    return cudaGetLastError();
}

}  // namespace sfcb200
