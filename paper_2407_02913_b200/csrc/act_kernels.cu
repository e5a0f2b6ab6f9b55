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

#include <mutex>

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

// `fused`: the staging area holds int16 V (kept across the grid barrier) instead of int8 vq.
template <int V, int CC>
__host__ __device__ inline ActSmem act_smem(int tw, bool fused) {
    using T = Tab<V>;
    ActSmem s;
    s.wcp = ((tw - 1) * T::M + T::n + 3) & ~3;
    s.chs = T::n * s.wcp;
    if (((s.chs / 4) & 1) == 0) s.chs += 4;
    s.x_off = 0;
    s.z_off = (size_t(s.chs) * CC + 15) & ~size_t(15);
    s.q_off = s.z_off + ((size_t(tw) * T::n * T::K * CC * 2 + 15) & ~size_t(15));
    s.bytes = s.q_off + size_t(tw) * T::F * CC * (fused ? 2 : 1);
    return s;
}
}  // namespace

// Grid-wide barrier for a co-resident (cooperatively launched) grid; called by ONE
// thread per CTA.  `bar[0]` counts arrivals and is reset by the last arriver, which
// then bumps the generation `bar[1]` the others spin on, so the pair is reusable
// without re-initialisation as long as bar[0] starts at 0.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
    const unsigned gen = ld_acquire(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
        atomicExch(bar, 0u);
        __threadfence();
        atomicAdd(bar + 1, 1u);
    } else {
        while (ld_acquire(bar + 1) == gen) __nanosleep(64);
    }
    __threadfence();
}

// MODE 0: max|V| -> atomicMax(*vmax).  MODE 1: quantize with the scale derived
// from *vmax_in and write vq[f][t][c] (row pitch Cpad) for f = k*K + l.
// MODE 2 (fused, co-resident grid only): V is computed once and kept in shared memory
// as int16 (|V| <= 4608), the block max goes to *vmax, a grid barrier publishes the
// global max, and the quantized rows are written from the kept V -- one launch and
// one transform instead of two of each.
template <int V, int MODE, int CC>
__global__ void __launch_bounds__(kActThreads) k_act(const int8_t* __restrict__ x, ConvGeom g,
                                                     int* __restrict__ vmax, const int* __restrict__ vmax_in, int bits,
                                                     QuantParams* __restrict__ qp_out, int8_t* __restrict__ vqA,
                                                     unsigned long long* __restrict__ sat, unsigned* __restrict__ gbar,
                                                     const QuantParams* __restrict__ qtab) {
    using T = Tab<V>;
    constexpr int n = T::n, K = T::K, M = T::M, F = T::F;
    constexpr int TPC = kActThreads / CC;   // work-groups per channel
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr int kTl = MODE == 0 ? kTlAbsmax : (MODE == 1 ? kTlQuant : kTlFused);
    tl_mark(kTl, 0);
    if (MODE == 0) griddep_launch_dependents();

    const int tw = g.tw;
    const int ti = blockIdx.x, b = blockIdx.y, c0 = blockIdx.z * CC;
    const int nch = min(CC, g.C - c0);
    const ActSmem L = act_smem<V, CC>(tw, MODE == 2);
    int8_t* s_x = reinterpret_cast<int8_t*>(smem + L.x_off);     // [CC][n][wcp], channel stride chs
    int16_t* s_z = reinterpret_cast<int16_t*>(smem + L.z_off);   // [tw][n][K][CC]
    int8_t* s_q = reinterpret_cast<int8_t*>(smem + L.q_off);     // [tw][F][CC]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = threadIdx.x % CC, j = threadIdx.x / CC;

    // ---- stage 0: stage rows [ih0, ih0 + n) of the CTA's channels as [c][r][pad + col],
    // zero outside the image.  A channel's window rows are one contiguous byte range of
    // NCHW (seg bytes), so the CTA moves 32-bit words: word w of channel ch covers bytes
    // [4w - mis, 4w - mis + 4) of the segment (mis = its start's misalignment); words fully
    // inside the segment are one LDG.32, the partial head / tail words byte loads.  A
    // thread derives (row, col) of its word's first byte once (multiply-high, exact for
    // i < 2^32 / W) and steps it.  The first batch of loads is in flight while the whole
    // staging area is zeroed with 16-byte stores.
    {
        const int ih0 = ti * M - g.pad;
        const int r_lo = max(ih0, 0), nrows = min(ih0 + n, g.H) - r_lo;
        const int rimg0 = r_lo - ih0;  // first staged row that holds image data
        const size_t cstride = size_t(g.H) * g.W;
        const int seg = nrows * g.W;
        const unsigned wmagic = 0xffffffffu / unsigned(g.W) + 1u;
        const int8_t* src0 = x + (size_t(b) * g.C + c0) * cstride + size_t(r_lo) * g.W;
        int8_t* dst0 = s_x + rimg0 * L.wcp + g.pad;
        const int nw = (seg + 6) >> 2;  // words covering seg bytes at any misalignment
        const unsigned nwmagic = 0xffffffffu / unsigned(nw) + 1u;
        const int total = nch * nw;
        constexpr int kJ = 4;
        uint32_t wv[kJ];
        int wch[kJ], wlo[kJ];
        auto load = [&](int k0) {
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj) {
                const int k = k0 + jj * kActThreads + int(threadIdx.x);
                wlo[jj] = 1 << 30;  // nothing to store
                if (k < total) {
                    const int ch = nw == 1 ? k : int(__umulhi(unsigned(k), nwmagic));
                    const int w = k - ch * nw;
                    const int8_t* cs = src0 + size_t(ch) * cstride;
                    const int mis = int(reinterpret_cast<uintptr_t>(cs) & 3);
                    const int lo = 4 * w - mis;  // segment index of the word's first byte
                    uint32_t v = 0;
                    if (lo >= 0 && lo + 4 <= seg) {
                        v = __ldg(reinterpret_cast<const unsigned int*>(cs + lo));
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (lo + q >= 0 && lo + q < seg) v |= uint32_t(uint8_t(__ldg(cs + lo + q))) << (8 * q);
                    }
                    wv[jj] = v, wch[jj] = ch, wlo[jj] = lo;
                }
            }
        };
        auto store = [&]() {
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj) {
                const int lo = wlo[jj];
                if (lo >= seg) continue;
                const int i0 = lo < 0 ? 0 : lo;  // first in-segment byte
                int r = g.W == 1 ? i0 : int(__umulhi(unsigned(i0), wmagic));
                int col = i0 - r * g.W;
                int8_t* d = dst0 + wch[jj] * L.chs;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = lo + q;
                    if (i < i0 || i >= seg) continue;
                    d[r * L.wcp + col] = int8_t(wv[jj] >> (8 * q));
                    if (++col == g.W) col = 0, ++r;
                }
            }
        };
        load(0);
        uint4* z4 = reinterpret_cast<uint4*>(s_x);
        for (int i = threadIdx.x; i < (L.chs * CC) / 16; i += kActThreads) z4[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        store();
        for (int k0 = kJ * kActThreads; k0 < total; k0 += kJ * kActThreads) {
            load(k0);
            store();
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

    if (MODE == 2) {
        int16_t* s_v = reinterpret_cast<int16_t*>(smem + L.q_off);  // [tw][F][CC]
        __shared__ int s_max;
        if (threadIdx.x == 0) s_max = 0;
        __syncthreads();
        int local = 0;
        for (int idx = j; idx < tw * K; idx += TPC) {
            const int l = idx % K, tj = idx / K;
            int zr[n];
#pragma unroll
            for (int r = 0; r < n; ++r) zr[r] = s_z[((tj * n + r) * K + l) * CC + c];
            int v[K];
            fwd1d<V>(zr, v);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                s_v[(tj * F + k * K + l) * CC + c] = int16_t(v[k]);
                local = max(local, abs(v[k]));
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
        if (lane == 0 && local > 0) atomicMax(&s_max, local);
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s_max > 0) atomicMax(vmax, s_max);
            grid_barrier(gbar, gridDim.x * gridDim.y * gridDim.z);
            s_max = int(ld_acquire(reinterpret_cast<const unsigned*>(vmax)));
        }
        __syncthreads();
        const QuantParams qp = qparams_for(s_max, bits, qtab);
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) *qp_out = qp;
        griddep_launch_dependents();  // every CTA is resident: the GEMM may start its prologue

        // quantize 4 channels per 32-bit word straight from the kept V
        constexpr int WPR = CC / 4;
        const int t0 = (b * g.th + ti) * tw;
        auto store = [&](auto quantize) {
            for (int i = threadIdx.x; i < tw * F * WPR; i += kActThreads) {
                const int wd = i % WPR, row = i / WPR;
                const int f = row % F, tj = row / F;
                const uint2 v4 = *reinterpret_cast<const uint2*>(s_v + size_t(row) * CC + wd * 4);
                const uint32_t q0 = uint32_t(quantize(int(int16_t(v4.x & 0xffff)))) & 0xff;
                const uint32_t q1 = uint32_t(quantize(int(v4.x) >> 16)) & 0xff;
                const uint32_t q2 = uint32_t(quantize(int(int16_t(v4.y & 0xffff)))) & 0xff;
                const uint32_t q3 = uint32_t(quantize(int(v4.y) >> 16)) & 0xff;
                reinterpret_cast<uint32_t*>(vqA + (size_t(f) * g.Tpad + t0 + tj) * g.Cpad + c0)[wd] =
                    q0 | (q1 << 8) | (q2 << 16) | (q3 << 24);
            }
        };
        if (qp.exact) {
            const long long mul = qp.mul, half = 1ll << (qp.shift - 1);
            const int shift = qp.shift;
            store([=](int v) { return int(((long long)v * mul + half) >> shift); });
        } else {
            store([&](int v) { return clamp_q(exact_q(v, qp.sa), qp.qmax, sat); });
        }
        tl_mark(kTl, 2);
        return;
    }

    QuantParams qp{};
    if (MODE == 1) {
        griddep_wait();  // the absmax pre-pass (and any multi-GPU MAX exchange) is complete
        tl_mark(kTl, 1);
        qp = qparams_for(*vmax_in, bits, qtab);
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) *qp_out = qp;
    }
    __syncthreads();  // stage 1's s_z is complete (the table lookup does not synchronise)

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
        griddep_wait();  // under PDL: *vmax has been zeroed by the predecessor
        tl_mark(kTl, 1);
        if (lane == 0 && local > 0) atomicMax(vmax, local);
        tl_mark(kTl, 2);
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
    tl_mark(kTl, 2);
}

// Stand-alone quantizer derivation (stats / the exhaustive test hook).
__global__ void k_quant_params(const int* __restrict__ vmax_p, int bits, QuantParams* __restrict__ qp,
                               unsigned long long* sat, const QuantParams* __restrict__ qtab) {
    const QuantParams p = qparams_for(*vmax_p, bits, qtab);
    if (threadIdx.x == 0) {
        *qp = p;
        *sat = 0;
    }
}

// One warp per table entry: bits = 2 + e / (kQpTableMax + 1), vmax = e % (kQpTableMax + 1).
__global__ void k_build_qtable(QuantParams* __restrict__ tab) {
    const int e = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (e >= kQpTableEntries) return;
    const QuantParams p = derive_qparams_warp(e % (kQpTableMax + 1), 2 + e / (kQpTableMax + 1));
    if ((threadIdx.x & 31) == 0) tab[e] = p;
}

__global__ void k_debug_quant(const QuantParams* __restrict__ qpp, int vmax, int32_t* __restrict__ q,
                              unsigned long long* sat) {
    const QuantParams qp = *qpp;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= 2 * vmax; i += gridDim.x * blockDim.x)
        q[i] = quant_act(i - vmax, qp, sat);
}

// ============================================================================ host
const QuantParams* qparams_table(bool build) {
    static std::mutex mu;
    static QuantParams* tabs[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (tabs[dev] || !build) return tabs[dev];
    std::lock_guard<std::mutex> lock(mu);
    if (tabs[dev]) return tabs[dev];
    QuantParams* t = nullptr;
    if (cudaMalloc(&t, sizeof(QuantParams) * kQpTableEntries) != cudaSuccess) return nullptr;
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return cudaFree(t), nullptr;
    k_build_qtable<<<(kQpTableEntries * 32 + 255) / 256, 256, 0, s>>>(t);
    const bool ok = cudaGetLastError() == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
    cudaStreamDestroy(s);
    if (!ok) return cudaFree(t), nullptr;
    tabs[dev] = t;
    return t;
}

namespace {

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// MODE 2 returns cudaErrorCooperativeLaunchTooLarge (nothing launched) when the grid
// cannot be co-resident; the caller then runs the two-kernel form.
template <int V, int MODE, int CC>
cudaError_t act_launch_cc(const int8_t* x, const ConvGeom& g, int* vmax, const int* vmax_in, int bits,
                          QuantParams* qp, int8_t* vqA, unsigned long long* sat, unsigned* gbar, cudaStream_t st,
                          bool pdl) {
    const size_t smem = act_smem<V, CC>(g.tw, MODE == 2).bytes;
    auto kern = k_act<V, MODE, CC>;
    static size_t attr_bytes = 0;  // per instantiation: raise the opt-in only when a layer needs more
    int per_sm = 0;
    if (smem > attr_bytes) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        attr_bytes = smem;
    }
    const long grid = long(g.th) * g.B * ((g.C + CC - 1) / CC);
    if (MODE == 2) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kActThreads, smem) != cudaSuccess)
            return cudaErrorCooperativeLaunchTooLarge;
        if (long(per_sm) * sm_count() < grid) return cudaErrorCooperativeLaunchTooLarge;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.th, g.B, (g.C + CC - 1) / CC);
    cfg.blockDim = dim3(kActThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (MODE == 2) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na++].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, x, g, vmax, vmax_in, bits, qp, vqA, sat, gbar,
                              MODE == 0 ? nullptr : qparams_table(false));
}

// Channels per CTA: 32 gives full 32-byte vq row segments; shrink for two waves
// over the 148 SMs and a <= 96 KB shared-memory footprint.
template <int V>
int pick_cc(const ConvGeom& g) {
    auto ctas = [&](int c) { return long(g.th) * g.B * ((g.C + c - 1) / c); };
    auto smem = [&](int c) {
        return c == 32 ? act_smem<V, 32>(g.tw, true).bytes
             : c == 16 ? act_smem<V, 16>(g.tw, true).bytes
             : c == 8  ? act_smem<V, 8>(g.tw, true).bytes
                       : act_smem<V, 4>(g.tw, true).bytes;
    };
    int cc = 32;
    while (cc > 4 && ctas(cc) < 2 * 148) cc /= 2;
    while (cc > 4 && smem(cc) > 96 * 1024) cc /= 2;
    return cc;
}

template <int V, int MODE>
cudaError_t act_launch(const int8_t* x, const ConvGeom& g, int* vmax, const int* vmax_in, int bits, QuantParams* qp,
                       int8_t* vqA, unsigned long long* sat, unsigned* gbar, cudaStream_t st, bool pdl) {
    switch (pick_cc<V>(g)) {
        case 32: return act_launch_cc<V, MODE, 32>(x, g, vmax, vmax_in, bits, qp, vqA, sat, gbar, st, pdl);
        case 16: return act_launch_cc<V, MODE, 16>(x, g, vmax, vmax_in, bits, qp, vqA, sat, gbar, st, pdl);
        case 8: return act_launch_cc<V, MODE, 8>(x, g, vmax, vmax_in, bits, qp, vqA, sat, gbar, st, pdl);
        default: return act_launch_cc<V, MODE, 4>(x, g, vmax, vmax_in, bits, qp, vqA, sat, gbar, st, pdl);
    }
}

}  // namespace

cudaError_t launch_act_absmax(int variant, const int8_t* x, const ConvGeom& g, int* vmax, cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return act_launch<0, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, nullptr, st, pdl);
        case 1: return act_launch<1, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, nullptr, st, pdl);
        default: return act_launch<2, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, nullptr, st, pdl);
    }
}

cudaError_t launch_act_quant(int variant, const int8_t* x, const ConvGeom& g, const int* vmax, int bits,
                             QuantParams* qp, int8_t* vqA, unsigned long long* sat, cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return act_launch<0, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, nullptr, st, pdl);
        case 1: return act_launch<1, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, nullptr, st, pdl);
        default: return act_launch<2, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, nullptr, st, pdl);
    }
}

cudaError_t launch_act_fused(int variant, const int8_t* x, const ConvGeom& g, int* vmax, int bits, QuantParams* qp,
                             int8_t* vqA, unsigned long long* sat, unsigned* gbar, cudaStream_t st) {
    switch (variant) {
        case 0: return act_launch<0, 2>(x, g, vmax, nullptr, bits, qp, vqA, sat, gbar, st, false);
        case 1: return act_launch<1, 2>(x, g, vmax, nullptr, bits, qp, vqA, sat, gbar, st, false);
        default: return act_launch<2, 2>(x, g, vmax, nullptr, bits, qp, vqA, sat, gbar, st, false);
    }
}

SFC_TL_UNIT_READER(tl_read_act)

cudaError_t launch_quant_params(const int* vmax, int bits, QuantParams* qp, unsigned long long* sat,
                                cudaStream_t st) {
    k_quant_params<<<1, 256, 0, st>>>(vmax, bits, qp, sat, qparams_table(false));
    return cudaGetLastError();
}

cudaError_t launch_debug_quant(const QuantParams* qp, int vmax, int32_t* q, unsigned long long* sat,
                               cudaStream_t st) {
    k_debug_quant<<<64, 256, 0, st>>>(qp, vmax, q, sat);
    return cudaGetLastError();
}

}  // namespace sfcb200
