// Stage 5 of the quantized SFC conv: the output transform with correction rows
// folded into A, in exact integers, then dequantisation / requantisation
// (reference: proj/src/quant.cpp:258-278).
//
// Persistent, TMA-fed: a block is (image b, tile row ti, TB tile columns, 32 output
// channels).  A producer warp streams the block's P slice P[0..F)[t0..t0+TB)[oc0..oc0+32)
// into shared memory with ONE 3-D TMA load (double-buffered, mbarrier handshake), and
// sixteen compute warps run
//   stage A  Q[t1][l]  = sum_k A[k][t1] P[k*K + l]      (scheduled inverse, transforms.cuh)
//   stage B  y[t1][t2] = sum_l Q[t1][l] A[l][t2]
//   stage C  output row segments (oc, oh, TB*M columns):  y_int, fp32 / fp64 y * sa * sf[oc] / N^2,
//            int8 clamp(rint(y * scale * s), 0, 127)
// Shared strides are odd so lanes stepping oc hit distinct banks.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"
#include "transforms.cuh"

namespace sfcb200 {

namespace {
constexpr int kOcc = 32;                     // output channels per block (128-byte TMA rows)
constexpr int kComputeWarps = 16;
constexpr int kOutThreads = 32 * (kComputeWarps + 1);

template <int V>
__host__ __device__ constexpr int out_tb() {  // tile columns per block: ~40 KB of P per block
    return (40 * 1024) / (Tab<V>::F * kOcc * 4) < 1 ? 1 : (40 * 1024) / (Tab<V>::F * kOcc * 4);
}

struct OutSmem {
    int qstride, ystride;
    size_t p_bytes, q_off, y_off, bar_off, bytes;
};

template <int V, bool Y64>
__host__ __device__ inline OutSmem out_smem() {
    using T = Tab<V>;
    constexpr int TB = out_tb<V>();
    const size_t es = Y64 ? 8 : 4;
    OutSmem s;
    s.qstride = kOcc | 1;
    s.ystride = (T::M * TB) | 1;
    s.p_bytes = size_t(T::F) * TB * kOcc * 4;
    s.q_off = 2 * s.p_bytes;
    s.y_off = (s.q_off + size_t(TB) * T::M * T::K * s.qstride * es + 15) & ~size_t(15);
    s.bar_off = (s.y_off + size_t(T::M) * kOcc * s.ystride * es + 15) & ~size_t(15);
    s.bytes = s.bar_off + 64;
    return s;
}

__device__ __forceinline__ void named_sync() {  // the compute warps only
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kComputeWarps) : "memory");
}
}  // namespace

template <int V, bool Y64>
__global__ void __launch_bounds__(kOutThreads, 1)
    k_output(const __grid_constant__ CUtensorMap tmP, ConvGeom g, const QuantParams* __restrict__ qpp,
             const double* __restrict__ sf, OutPtrs o) {
    using T = Tab<V>;
    constexpr int K = T::K, M = T::M, F = T::F, TB = out_tb<V>();
    using acc_t = typename std::conditional<Y64, long long, int>::type;
    extern __shared__ __align__(128) uint8_t smem[];
    const OutSmem L = out_smem<V, Y64>();
    acc_t* s_q = reinterpret_cast<acc_t*>(smem + L.q_off);   // [TB][M][K] rows of qstride
    acc_t* s_y = reinterpret_cast<acc_t*>(smem + L.y_off);   // [M][kOcc] rows of ystride
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + 2;
    __shared__ double s_scale[kOcc];

    const int tcols = (g.tw + TB - 1) / TB, ocb = (g.OC + kOcc - 1) / kOcc;
    const int blocks = g.B * g.th * tcols * ocb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], kComputeWarps);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    griddep_wait();  // P complete
    griddep_launch_dependents();

    if (warp == kComputeWarps) {  // ---- producer
        if (lane == 0) {
            ptx::tma_prefetch(&tmP);
            int i = 0;
            for (int blk = blockIdx.x; blk < blocks; blk += gridDim.x, ++i) {
                const int buf = i & 1;
                ptx::mbar_wait(&empty[buf], ((i >> 1) & 1) ^ 1);
                const int oc0 = (blk % ocb) * kOcc, rest = blk / ocb;
                const int tc = rest % tcols, row = rest / tcols;  // row = b * th + ti
                ptx::mbar_expect_tx(&full[buf], uint32_t(L.p_bytes));
                ptx::tma_load_3d(smem + buf * L.p_bytes, &tmP, &full[buf], oc0, row * g.tw + tc * TB, 0);
            }
        }
        return;
    }

    // ---- compute warps
    const int WO = g.WO;
    int i = 0;
    for (int blk = blockIdx.x; blk < blocks; blk += gridDim.x, ++i) {
        const int buf = i & 1;
        const int oc0 = (blk % ocb) * kOcc, rest = blk / ocb;
        const int tc = rest % tcols, row = rest / tcols;
        const int b = row / g.th, ti = row % g.th;
        const int noc = min(kOcc, g.OC - oc0);
        const int ntb = min(TB, g.tw - tc * TB);
        if (threadIdx.x < kOcc && int(threadIdx.x) < noc)
            s_scale[threadIdx.x] = (qpp->sa * sf[oc0 + threadIdx.x]) / double(T::DEN * T::DEN);
        ptx::mbar_wait(&full[buf], (i >> 1) & 1);
        const int32_t* sp = reinterpret_cast<const int32_t*>(smem + buf * L.p_bytes);  // [F][TB][kOcc]

        // stage A: items (tj, l, oc)
        for (int it = threadIdx.x; it < TB * K * kOcc; it += 32 * kComputeWarps) {
            const int oc = it % kOcc, l = (it / kOcc) % K, tj = it / (kOcc * K);
            if (tj >= ntb) continue;
            acc_t pk[K], qt[M];
#pragma unroll
            for (int k = 0; k < K; ++k) pk[k] = sp[((k * K + l) * TB + tj) * kOcc + oc];
            inv1d<V>(pk, qt);
#pragma unroll
            for (int t1 = 0; t1 < M; ++t1) s_q[((tj * M + t1) * K + l) * L.qstride + oc] = qt[t1];
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[buf]);  // P buffer consumed: the producer may refill it
        named_sync();

        // stage B: items (tj, t1, oc)
        for (int it = threadIdx.x; it < TB * M * kOcc; it += 32 * kComputeWarps) {
            const int oc = it % kOcc, t1 = (it / kOcc) % M, tj = it / (kOcc * M);
            if (tj >= ntb) continue;
            acc_t qv[K], yt[M];
#pragma unroll
            for (int l = 0; l < K; ++l) qv[l] = s_q[((tj * M + t1) * K + l) * L.qstride + oc];
            inv1d<V>(qv, yt);
            acc_t* dst = s_y + (t1 * kOcc + oc) * L.ystride + tj * M;
#pragma unroll
            for (int t2 = 0; t2 < M; ++t2) dst[t2] = yt[t2];
        }
        named_sync();

        // stage C: the block's output row segments (t1, oc) x ncol columns, one element per
        // thread per pass (consecutive threads -> consecutive columns of a row); e / ncol by
        // multiply-high with a per-block magic, all offsets 32-bit relative to the block base.
        const int col0 = tc * TB * M;
        const int ncol = min(ntb * M, WO - col0);
        const int hrows = min(M, g.HO - ti * M);
        const unsigned magic = 0xffffffffu / unsigned(ncol) + 1u;
        const int total = M * kOcc * ncol;
        const int plane = g.HO * WO;
        const size_t base0 = (size_t(b) * g.OC + oc0) * size_t(plane) + size_t(ti) * M * WO + col0;
        auto emit = [&](auto store) {
            for (int e = threadIdx.x; e < total; e += 32 * kComputeWarps) {
                const int r = ncol == 1 ? e : int(__umulhi(unsigned(e), magic));
                const int c = e - r * ncol;
                const int oc = r % kOcc, t1 = r / kOcc;
                if (oc >= noc || t1 >= hrows) continue;
                store(base0 + unsigned(oc * plane + t1 * WO + c), s_y[r * L.ystride + c], s_scale[oc]);
            }
        };
        if (o.y32) emit([&](size_t x, acc_t y, double) { o.y32[x] = int(y); });
        if (o.y64) emit([&](size_t x, acc_t y, double) { o.y64[x] = (long long)y; });
        if (o.f32)
            emit([&](size_t x, acc_t y, double s) {
                o.f32[x] = Y64 ? float(double(y) * s) : __int2float_rn(int(y)) * float(s);
            });
        if (o.f64) emit([&](size_t x, acc_t y, double s) { o.f64[x] = double(y) * s; });
        if (o.i8)
            emit([&](size_t x, acc_t y, double s) {
                o.i8[x] = int8_t(fmin(fmax(rint(double(y) * s * o.requant), 0.0), 127.0));
            });
        named_sync();  // s_q / s_y / s_scale are rewritten by the next block
    }
}

namespace {
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

template <int V, bool Y64>
cudaError_t out_launch(const int32_t* P, const ConvGeom& g, const QuantParams* qp, const double* sf, const OutPtrs& o,
                       cudaStream_t st, bool pdl) {
    constexpr int TB = out_tb<V>();
    auto fn = encode_fn();
    if (!fn) return cudaErrorInvalidValue;
    CUtensorMap tm;
    cuuint64_t dims[3] = {cuuint64_t(g.OCpad), cuuint64_t(g.Tpad), cuuint64_t(Tab<V>::F)};
    cuuint64_t strides[2] = {cuuint64_t(g.OCpad) * 4, cuuint64_t(g.OCpad) * g.Tpad * 4};
    cuuint32_t box[3] = {kOcc, TB, Tab<V>::F};
    cuuint32_t estr[3] = {1, 1, 1};
    if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, const_cast<int32_t*>(P), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    const size_t smem = out_smem<V, Y64>().bytes;
    auto kern = k_output<V, Y64>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const long blocks = long(g.B) * g.th * ((g.tw + TB - 1) / TB) * ((g.OC + kOcc - 1) / kOcc);
    const int per_sm = int((227 * 1024) / (smem + 1024)) < 1 ? 1 : int((227 * 1024) / (smem + 1024));
    const long resident = long(sm_count()) * (per_sm > 2 ? 2 : per_sm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(blocks < resident ? blocks : resident));
    cfg.blockDim = dim3(kOutThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, tm, g, qp, sf, o);
}

template <int V>
cudaError_t out_by_width(bool y64, const int32_t* P, const ConvGeom& g, const QuantParams* qp, const double* sf,
                         const OutPtrs& o, cudaStream_t st, bool pdl) {
    return y64 ? out_launch<V, true>(P, g, qp, sf, o, st, pdl) : out_launch<V, false>(P, g, qp, sf, o, st, pdl);
}
}  // namespace

cudaError_t launch_output(int variant, bool y64, const int32_t* P, const ConvGeom& g, const QuantParams* qp,
                          const double* sf, const OutPtrs& o, cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return out_by_width<0>(y64, P, g, qp, sf, o, st, pdl);
        case 1: return out_by_width<1>(y64, P, g, qp, sf, o, st, pdl);
        default: return out_by_width<2>(y64, P, g, qp, sf, o, st, pdl);
    }
}

}  // namespace sfcb200
