// Stage 5 of the quantized SFC conv: the output transform with correction rows
// folded into A, in exact integers, then dequantisation / requantisation
// (reference: proj/src/quant.cpp:258-278).
//
//   stage A  Q[t1][l]  = sum_k A[k][t1] P[k*K + l]     items (tj, l, oc)
//   stage B  y[t1][t2] = sum_l Q[t1][l] A[l][t2]       items (tj, t1, oc) -> shared row tile
//   stage C  whole output rows (oc, oh) of the tile row, coalesced:
//            y_int, out = y * sa * sf[oc] / N^2 (fp32), out_i8 = clamp(rint(y * scale * s), 0, 127)
//
// One CTA per (image b, tile row ti, chunk of OCC output channels).  P reads are
// coalesced over oc; shared strides are odd so lanes stepping oc hit distinct banks.
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"
#include "transforms.cuh"

namespace sfcb200 {

namespace {
constexpr int kOutThreads = 256;

struct OutSmem {
    int qstride;   // elements per (tj, t1, l) row of Q  (>= OCC, odd)
    int ystride;   // elements per (t1, oc) output row   (>= M*tw, odd)
    size_t y_off, bytes;
};

template <int V, bool Y64, int OCC>
__host__ __device__ inline OutSmem out_smem(int tw) {
    using T = Tab<V>;
    const size_t es = Y64 ? 8 : 4;
    OutSmem s;
    s.qstride = OCC | 1;
    s.ystride = (T::M * tw) | 1;
    const size_t q = size_t(tw) * T::M * T::K * s.qstride * es;
    s.y_off = (q + 15) & ~size_t(15);
    s.bytes = s.y_off + size_t(T::M) * OCC * s.ystride * es;
    return s;
}
}  // namespace

template <int V, bool Y64, int OCC>
__global__ void __launch_bounds__(kOutThreads) k_output(const int32_t* __restrict__ P, ConvGeom g,
                                                        const QuantParams* __restrict__ qpp,
                                                        const double* __restrict__ sf, OutPtrs o) {
    using T = Tab<V>;
    constexpr int K = T::K, M = T::M;
    using acc_t = typename std::conditional<Y64, long long, int>::type;
    extern __shared__ __align__(16) uint8_t smem[];
    const int tw = g.tw;
    const OutSmem L = out_smem<V, Y64, OCC>(tw);
    acc_t* s_q = reinterpret_cast<acc_t*>(smem);            // [tw][M][K] rows of qstride
    acc_t* s_y = reinterpret_cast<acc_t*>(smem + L.y_off);  // [M][OCC] rows of ystride
    const int ti = blockIdx.x, b = blockIdx.y, oc0 = blockIdx.z * OCC;
    const int noc = min(OCC, g.OC - oc0);
    const int t0 = (b * g.th + ti) * tw;
    griddep_wait();  // P complete
    griddep_launch_dependents();

    // ---- stage A
    for (int it = threadIdx.x; it < tw * K * OCC; it += kOutThreads) {
        const int oc = it % OCC, l = (it / OCC) % K, tj = it / (OCC * K);
        if (oc >= noc) continue;
        const int32_t* src = P + (size_t(l) * g.Tpad + t0 + tj) * g.OCpad + oc0 + oc;
        int p[K];
#pragma unroll
        for (int k = 0; k < K; ++k) p[k] = __ldg(src + size_t(k) * K * g.Tpad * g.OCpad);
        acc_t pk[K], qt[M];
#pragma unroll
        for (int k = 0; k < K; ++k) pk[k] = p[k];
        inv1d<V>(pk, qt);
#pragma unroll
        for (int t1 = 0; t1 < M; ++t1) s_q[((tj * M + t1) * K + l) * L.qstride + oc] = qt[t1];
    }
    __syncthreads();

    // ---- stage B
    for (int it = threadIdx.x; it < tw * M * OCC; it += kOutThreads) {
        const int oc = it % OCC, t1 = (it / OCC) % M, tj = it / (OCC * M);
        if (oc >= noc) continue;
        acc_t qv[K];
#pragma unroll
        for (int l = 0; l < K; ++l) qv[l] = s_q[((tj * M + t1) * K + l) * L.qstride + oc];
        acc_t* dst = s_y + (t1 * OCC + oc) * L.ystride + tj * M;
        acc_t yt[M];
        inv1d<V>(qv, yt);
#pragma unroll
        for (int t2 = 0; t2 < M; ++t2) dst[t2] = yt[t2];
    }
    __syncthreads();

    // ---- stage C: one warp per output row (t1, oc), lanes along ow
    __shared__ double s_scale[OCC];
    if (threadIdx.x < OCC && int(threadIdx.x) < noc)
        s_scale[threadIdx.x] = (qpp->sa * sf[oc0 + threadIdx.x]) / double(T::DEN * T::DEN);
    __syncthreads();
    // Rows of at most 32 columns are packed several per warp (lane -> (sub-row, ow)); one
    // tight loop per requested output so no per-element pointer tests remain.
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int WO = g.WO;
    const int rpw = WO <= 32 ? 32 / WO : 1;       // rows per warp pass
    const int sub = WO <= 32 ? lane / WO : 0;
    const int col0 = WO <= 32 ? lane % WO : lane;
    const int cstep = WO <= 32 ? 32 : 32;          // only used when WO > 32
    const bool lane_ok = sub < rpw;
    const int hrows = min(M, g.HO - ti * M);       // output rows of this tile row inside the image
    const size_t plane = size_t(g.HO) * WO;
    const size_t base0 = (size_t(b) * g.OC + oc0) * plane + size_t(ti) * M * WO;
    auto emit = [&](auto store) {
        for (int r0 = warp * rpw; r0 < M * OCC; r0 += (kOutThreads / 32) * rpw) {
            const int row = r0 + sub;
            const int oc = row % OCC, t1 = row / OCC;
            if (!lane_ok || row >= M * OCC || oc >= noc || t1 >= hrows) continue;
            const acc_t* src = s_y + (t1 * OCC + oc) * L.ystride;
            const size_t base = base0 + oc * plane + t1 * WO;
            const double scale = s_scale[oc];
            for (int c = col0; c < WO; c += (WO <= 32 ? 1 << 30 : cstep)) store(base + c, src[c], scale);
        }
    };
    if (o.y32) emit([&](size_t i, acc_t y, double) { o.y32[i] = int(y); });
    if (o.y64) emit([&](size_t i, acc_t y, double) { o.y64[i] = (long long)y; });
    if (o.f32)
        emit([&](size_t i, acc_t y, double s) {
            o.f32[i] = Y64 ? float(double(y) * s) : __int2float_rn(int(y)) * float(s);
        });
    if (o.f64) emit([&](size_t i, acc_t y, double s) { o.f64[i] = double(y) * s; });
    if (o.i8)
        emit([&](size_t i, acc_t y, double s) {
            o.i8[i] = int8_t(fmin(fmax(rint(double(y) * s * o.requant), 0.0), 127.0));
        });
}

namespace {
template <int V, bool Y64, int OCC>
cudaError_t out_launch_occ(const int32_t* P, const ConvGeom& g, const QuantParams* qp, const double* sf, const OutPtrs& o, cudaStream_t st,
                           bool pdl) {
    const size_t smem = out_smem<V, Y64, OCC>(g.tw).bytes;
    auto kern = k_output<V, Y64, OCC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.th, g.B, (g.OC + OCC - 1) / OCC);
    cfg.blockDim = dim3(kOutThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, P, g, qp, sf, o);
}

template <int V, bool Y64>
cudaError_t out_launch(const int32_t* P, const ConvGeom& g, const QuantParams* qp, const double* sf, const OutPtrs& o, cudaStream_t st, bool pdl) {
    auto ctas = [&](int o) { return long(g.th) * g.B * ((g.OC + o - 1) / o); };
    auto smem = [&](int o) {
        return o == 32 ? out_smem<V, Y64, 32>(g.tw).bytes
             : o == 16 ? out_smem<V, Y64, 16>(g.tw).bytes
             : o == 8  ? out_smem<V, Y64, 8>(g.tw).bytes
                       : out_smem<V, Y64, 4>(g.tw).bytes;
    };
    int occ = 32;
    while (occ > 4 && ctas(occ) < 2 * 148) occ /= 2;
    while (occ > 4 && smem(occ) > 96 * 1024) occ /= 2;
    switch (occ) {
        case 32: return out_launch_occ<V, Y64, 32>(P, g, qp, sf, o, st, pdl);
        case 16: return out_launch_occ<V, Y64, 16>(P, g, qp, sf, o, st, pdl);
        case 8: return out_launch_occ<V, Y64, 8>(P, g, qp, sf, o, st, pdl);
        default: return out_launch_occ<V, Y64, 4>(P, g, qp, sf, o, st, pdl);
    }
}

template <int V>
cudaError_t out_by_width(bool y64, const int32_t* P, const ConvGeom& g, const QuantParams* qp, const double* sf, const OutPtrs& o, cudaStream_t st,
                         bool pdl) {
    return y64 ? out_launch<V, true>(P, g, qp, sf, o, st, pdl)
               : out_launch<V, false>(P, g, qp, sf, o, st, pdl);
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
