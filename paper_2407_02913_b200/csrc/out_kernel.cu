// Stage 5 of the quantized SFC conv: the output transform with correction rows
// folded into A, in exact integers, then dequantisation / requantisation
// (reference: proj/src/quant.cpp:258-278).
//
// One CTA per block: a block is (image b, tile row ti, TB tile columns, 32 output
// channels).  Thread 0 brings the block's P slice P[0..F)[t0..t0+TB)[oc0..oc0+32) into
// shared memory with ONE 3-D TMA load (mbarrier completion), then sixteen warps run
//   stage A  Q[t1][l]  = sum_k A[k][t1] P[k*K + l]      (scheduled inverse, transforms.cuh)
//   stage B  y[t1][t2] = sum_l Q[t1][l] A[l][t2]         (y overwrites the consumed P slice)
//   stage C  output row segments (oc, oh, TB*M columns), all requested outputs in one pass:
//            y_int, fp32 / fp64 y * sa * sf[oc] / N^2, int8 clamp(rint(y * scale * s), 0, 127)
// Not persistent: a CTA needs ~62 KB, so two or three are resident per SM and hide each
// other's TMA / barrier latency (the persistent double-buffered form needed 115 KB and ran
// one CTA per SM at 25% warp occupancy on the 28x28 layers).  Shared strides are odd so
// lanes stepping oc hit distinct banks.
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
constexpr int kOcc = 32;  // output channels per block (128-byte TMA rows)
constexpr int kOutThreads = 512;

template <int V>
__host__ __device__ constexpr int out_tb() {  // tile columns per block: ~40 KB of P per block
    return (40 * 1024) / (Tab<V>::F * kOcc * 4) < 1 ? 1 : (40 * 1024) / (Tab<V>::F * kOcc * 4);
}

struct OutSmem {
    int qstride, ystride;
    size_t p_bytes, q_off, bar_off, bytes;
};

template <int V, bool Y64>
__host__ __device__ inline OutSmem out_smem() {
    using T = Tab<V>;
    constexpr int TB = out_tb<V>();
    const size_t es = Y64 ? 8 : 4;
    OutSmem s;
    s.qstride = kOcc | 1;
    s.ystride = (T::M * TB) | 1;
    const size_t y_bytes = size_t(T::M) * kOcc * s.ystride * es;
    s.p_bytes = size_t(T::F) * TB * kOcc * 4;
    if (y_bytes > s.p_bytes) s.p_bytes = y_bytes;  // s_y reuses the P slice
    s.q_off = (s.p_bytes + 127) & ~size_t(127);
    s.bar_off = (s.q_off + size_t(TB) * T::M * T::K * s.qstride * es + 15) & ~size_t(15);
    s.bytes = s.bar_off + 16;
    return s;
}
}  // namespace

template <int V, bool Y64>
__global__ void __launch_bounds__(kOutThreads, 2)
    k_output(const __grid_constant__ CUtensorMap tmP, ConvGeom g, const QuantParams* __restrict__ qpp,
             const double* __restrict__ sf, OutPtrs o) {
    using T = Tab<V>;
    constexpr int K = T::K, M = T::M, TB = out_tb<V>();
    using acc_t = typename std::conditional<Y64, long long, int>::type;
    extern __shared__ __align__(128) uint8_t smem[];
    const OutSmem L = out_smem<V, Y64>();
    const int32_t* sp = reinterpret_cast<const int32_t*>(smem);  // [F][TB][kOcc]
    acc_t* s_y = reinterpret_cast<acc_t*>(smem);                 // [M][kOcc] rows of ystride (after stage A)
    acc_t* s_q = reinterpret_cast<acc_t*>(smem + L.q_off);       // [TB][M][K] rows of qstride
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    __shared__ double s_scale[kOcc];

    const int tcols = (g.tw + TB - 1) / TB, ocb = (g.OC + kOcc - 1) / kOcc;
    const int blk = blockIdx.x;
    tl_mark(kTlOutput, 0);
    const int oc0 = (blk % ocb) * kOcc, rest = blk / ocb;
    const int tc = rest % tcols, row = rest / tcols;  // row = b * th + ti
    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tmP);
        ptx::mbar_init(full, 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    griddep_wait();  // P complete
    tl_mark(kTlOutput, 1);
    griddep_launch_dependents();
    if (threadIdx.x == 0) {
        ptx::mbar_expect_tx(full, uint32_t(size_t(T::F) * TB * kOcc * 4));
        ptx::tma_load_3d(smem, &tmP, full, oc0, row * g.tw + tc * TB, 0);
    }
    const int b = row / g.th, ti = row % g.th;
    const int noc = min(kOcc, g.OC - oc0);
    const int ntb = min(TB, g.tw - tc * TB);
    if (threadIdx.x < kOcc && int(threadIdx.x) < noc)
        s_scale[threadIdx.x] = (qpp->sa * sf[oc0 + threadIdx.x]) / double(T::DEN * T::DEN);
    ptx::mbar_wait(full, 0);

    // stage A: items (tj, l, oc)
    for (int it = threadIdx.x; it < TB * K * kOcc; it += kOutThreads) {
        const int oc = it % kOcc, l = (it / kOcc) % K, tj = it / (kOcc * K);
        if (tj >= ntb) continue;
        acc_t pk[K], qt[M];
#pragma unroll
        for (int k = 0; k < K; ++k) pk[k] = sp[((k * K + l) * TB + tj) * kOcc + oc];
        inv1d<V>(pk, qt);
#pragma unroll
        for (int t1 = 0; t1 < M; ++t1) s_q[((tj * M + t1) * K + l) * L.qstride + oc] = qt[t1];
    }
    __syncthreads();

    // stage B: items (tj, t1, oc)
    for (int it = threadIdx.x; it < TB * M * kOcc; it += kOutThreads) {
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
    __syncthreads();

    // stage C: the block's output row segments (t1, oc) x ncol columns, one element per
    // thread per pass (consecutive threads -> consecutive columns of a row); e / ncol by
    // multiply-high with a per-block magic, all offsets 32-bit relative to the block base.
    const int WO = g.WO;
    const int col0 = tc * TB * M;
    const int ncol = min(ntb * M, WO - col0);
    const int hrows = min(M, g.HO - ti * M);
    const unsigned magic = 0xffffffffu / unsigned(ncol) + 1u;
    const int total = M * kOcc * ncol;
    const int plane = g.HO * WO;
    const size_t base0 = (size_t(b) * g.OC + oc0) * size_t(plane) + size_t(ti) * M * WO + col0;
    int* const y32 = o.y32 ? o.y32 + base0 : nullptr;
    int64_t* const y64 = o.y64 ? o.y64 + base0 : nullptr;
    float* const f32 = o.f32 ? o.f32 + base0 : nullptr;
    double* const f64 = o.f64 ? o.f64 + base0 : nullptr;
    int8_t* const i8 = o.i8 ? o.i8 + base0 : nullptr;
    const double rq = o.requant;
    for (int e = threadIdx.x; e < total; e += kOutThreads) {
        const int r = ncol == 1 ? e : int(__umulhi(unsigned(e), magic));
        const int c = e - r * ncol;
        const int oc = r % kOcc, t1 = r / kOcc;
        if (oc >= noc || t1 >= hrows) continue;
        const unsigned x = unsigned(oc * plane + t1 * WO + c);
        const acc_t y = s_y[r * L.ystride + c];
        if (y32) y32[x] = int(y);
        if (y64) y64[x] = int64_t(y);
        if (f32 || f64 || i8) {
            const double s = s_scale[oc];
            if (f32) f32[x] = Y64 ? float(double(y) * s) : __int2float_rn(int(y)) * float(s);
            if (f64) f64[x] = double(y) * s;
            if (i8) i8[x] = int8_t(fmin(fmax(rint(double(y) * s * rq), 0.0), 127.0));
        }
    }
    __syncthreads();
    tl_mark(kTlOutput, 2);
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
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(blocks));
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

SFC_TL_UNIT_READER(tl_read_out)

cudaError_t launch_output(int variant, bool y64, const int32_t* P, const ConvGeom& g, const QuantParams* qp,
                          const double* sf, const OutPtrs& o, cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return out_by_width<0>(y64, P, g, qp, sf, o, st, pdl);
        case 1: return out_by_width<1>(y64, P, g, qp, sf, o, st, pdl);
        default: return out_by_width<2>(y64, P, g, qp, sf, o, st, pdl);
    }
}

}  // namespace sfcb200
