// Stage 5 of the quantized SFC conv on the tensor cores: the output transform with its
// correction rows (quant.cpp:264-278 with A from the spec, corrections folded into A),
//
//     y[t1][t2] = sum_{k,l} A[k][t1] A[l][t2] P[k*K + l]     (exact integers, y_int),
//
// is, per (tile, output channel) pair, a linear map of the pair's F transform-domain sums onto
// its M*M outputs with small integer coefficients W[(t1,t2)][(k,l)] = A[k][t1] A[l][t2]
// (|W| <= 36).  Over 128 pairs it is a GEMM  Y[128 x M^2] = P[128 x F] . W^T,  and with P split
// into its three bytes (P = b0 + 2^8 b1 + 2^16 b2, b0 / b1 unsigned, b2 signed: the 24-bit P
// of every BASELINE layer) it is three int8 GEMMs on tcgen05 (kind::i8, int32 accumulators in
// TMEM):  y = D0 + 2^8 D1 + 2^16 D2  (mod 2^32, exact because |y| < 2^31).  The CUDA-core
// inverse passes of out_kernel.cu (~400 dependent integer ops per pair) become 3 * ceil(F/32)
// MMAs per 128 pairs; the kernel is bound by the P bytes it streams.
//
// P arrives unit-major and pre-swizzled from the GEMM epilogue (sfc_kernels.hpp pu_offset):
// a unit = 32 output channels x 4 consecutive tiles = the 128 MMA rows; each byte plane is an
// MN-major A operand [F rows][128 B] in the 128B-swizzle pattern, fetched with one TMA box per
// plane.  B = W is K-major in shared memory, built once per CTA.
//
// Warp roles (persistent, one CTA per SM): 0 = TMA producer (2-3 stages), 1 = MMA issuer
// and TMEM owner (accumulators double-buffered: unit i+1's MMAs overlap unit i's epilogue),
// 2..13 = epilogue: warp w reads TMEM lane quarter w % 4 (= tile w % 4 of the unit, lane = oc)
// and part (w - 2) / 4 of the outputs, recombines the three planes, parks y in shared memory
// (double-buffered: one barrier per unit), then all 384 epilogue threads write the unit's
// output rows (4 tiles x M columns per row when the tiles share an image row) with the
// requested conversions.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "devcache.hpp"
#include "ptx.cuh"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"

namespace sfcb200 {

namespace {
constexpr int kOmParts = 3;                      // epilogue warps per TMEM lane quarter (output parts)
constexpr int kOmEpiWarps = 4 * kOmParts;
constexpr int kOmThreads = 64 + 32 * kOmEpiWarps;
constexpr int kOmMaxOc = 1024;  // per-channel scales kept in shared memory

template <int V>
struct Om {
    static constexpr int F = Tab<V>::F, K = Tab<V>::K, M = Tab<V>::M, MM = M * M;
    static constexpr int KP = (F + 31) / 32 * 32;      // frequencies padded to the MMA K step
    static constexpr int KB = (KP + 127) / 128;        // 128-byte K blocks of W
    static constexpr int PART = (MM + kOmParts - 1) / kOmParts;  // outputs per epilogue part (last: the rest)
    static constexpr int NP = (PART + 7) / 8 * 8;      // W rows (TMEM columns) per part
    static constexpr int N = (kOmParts * NP + 15) / 16 * 16;  // MMA N: 32 / 48 / 80
    static constexpr uint32_t PLANE = uint32_t(KP) * 128;
    static constexpr uint32_t STAGE = 3 * PLANE;
    static constexpr int STAGES = STAGE * 3 <= 150 * 1024 ? 3 : 2;  // bulk-copy pipeline depth
    static constexpr int ROW = kUnitTiles * M;         // staged columns per (oc, t1): 4 tiles x M
    static constexpr int OCS = M * ROW + 2;            // staged words per output channel, at most (see k_out_mma)
    static constexpr int TMEM_COLS = 6 * N <= 128 ? 128 : (6 * N <= 256 ? 256 : 512);
    static_assert(6 * N <= 512, "two buffers of three accumulators must fit TMEM");
    static constexpr size_t W_BYTES = size_t(KB) * N * 128;
    static constexpr size_t Y_BYTES = size_t(kUnitOc) * OCS * 4;  // one staging buffer (two are used)
    static constexpr size_t SMEM = 1024 + STAGES * size_t(STAGE) + W_BYTES + 2 * Y_BYTES + kOmMaxOc * 16 + 512;
};

struct TileInfo {
    long long base;  // output offset of the tile's (oc 0, t1 0, t2 0) element (channel oc0 of the unit)
    int rows, cols;  // valid output rows / columns (0 rows: padding tile)
};

__device__ __forceinline__ void named_bar_epi() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kOmEpiWarps) : "memory"); }

// MK: compile-time output set (bits: 1 y32, 2 y64, 4 f32, 8 f64, 16 i8); 0 = read o at run time
template <int V, int MK>
__global__ void __launch_bounds__(kOmThreads, 1)
    k_out_mma(const __grid_constant__ CUtensorMap tmP, ConvGeom g, const QuantParams* __restrict__ qpp,
              const double* __restrict__ sf, OutPtrs o, int n_ob, int n_tg, int units) {
    using C = Om<V>;
    using T = Tab<V>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned base, derived by pointer arithmetic so the compiler keeps shared accesses
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                                   // [stages][3 planes][KP rows][128 B]
    uint8_t* sW = sA + C::STAGES * size_t(C::STAGE);      // [KB][N rows][128 B], 128B-swizzled K-major
    int* s_y = reinterpret_cast<int*>(sW + C::W_BYTES);   // 2 x [32 oc][M rows][ROW] (row stride OCS per oc)
    double* s_scale = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(s_y) + 2 * C::Y_BYTES);
    float* s_scalef = reinterpret_cast<float*>(s_scale + kOmMaxOc);
    uint64_t* full = reinterpret_cast<uint64_t*>(s_scalef + kOmMaxOc);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    TileInfo* s_tile = reinterpret_cast<TileInfo*>(tempty + 2);  // 2 x [kUnitTiles]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_tile + 2 * kUnitTiles);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    tl_mark(kTlOutput, 0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) ptx::mbar_init(&full[s], 1), ptx::mbar_init(&empty[s], 1);
        for (int i = 0; i < 2; ++i) ptx::mbar_init(&tfull[i], 1), ptx::mbar_init(&tempty[i], kOmEpiWarps);
        ptx::fence_mbar_init();
    }
    // W rows n: part p = n / NP, output o = p * PART + n % NP (rows past the part's outputs and
    // columns f >= F are zero); byte f of row n at K block f / 128, chunk ((f % 128) / 16) ^ (n & 7)
    for (int i = threadIdx.x; i < C::KB * C::N * 128; i += kOmThreads) {
        const int kb = i / (C::N * 128), n = (i / 128) % C::N, b = i % 128;
        const int f = kb * 128 + b, pp = n / C::NP, idx = n % C::NP;
        int w = 0;
        if (pp < kOmParts && idx < C::PART && pp * C::PART + idx < C::MM && f < C::F) {
            const int oo = pp * C::PART + idx, t1 = oo / C::M, t2 = oo % C::M;
            w = T::a(f / C::K, t1) * T::a(f % C::K, t2);
        }
        sW[size_t(kb) * C::N * 128 + n * 128 + ((((b >> 4) ^ (n & 7)) << 4) | (b & 15))] = uint8_t(int8_t(w));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // W (generic stores) -> tensor core
    if (warp == 1) ptx::tmem_alloc(tmem_holder, C::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    griddep_wait();  // P and the activation scale are complete
    tl_mark(kTlOutput, 1);
    griddep_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            ptx::tma_prefetch(&tmP);
            int stage = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int ob = u % n_ob, tg = u / n_ob;
                ptx::mbar_wait_sleep(&empty[stage], phase ^ 1);
                ptx::mbar_expect_tx(&full[stage], 3u * C::F * 128);
                uint8_t* dst = sA + size_t(stage) * C::STAGE;
#pragma unroll
                for (int pl = 0; pl < 3; ++pl) ptx::tma_load_5d(dst + pl * C::PLANE, &tmP, &full[stage], 0, tg, 0, pl, ob);
                if (++stage == C::STAGES) stage = 0, phase ^= 1;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id_u = ptx::idesc_i8_amn(128, C::N, false), id_s = ptx::idesc_i8_amn(128, C::N, true);
            int stage = 0;
            uint32_t phase = 0;
            int i = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
                const int ab = i & 1;
                ptx::mbar_wait_sleep(&tempty[ab], ((i >> 1) & 1) ^ 1);
                ptx::mbar_wait_sleep(&full[stage], phase);
                ptx::tc_fence_after();
                const uint32_t a0 = ptx::smem_u32(sA + size_t(stage) * C::STAGE), w0 = ptx::smem_u32(sW);
#pragma unroll
                for (int ks = 0; ks < C::KP / 32; ++ks) {
                    const uint64_t bd = ptx::smem_desc_kmajor(w0 + (ks / 4) * (C::N * 128) + (ks % 4) * 32, 128);
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl)
                        ptx::mma_i8(tmem + uint32_t(ab * 3 * C::N + pl * C::N),
                                    ptx::smem_desc_mn128(a0 + pl * C::PLANE + ks * 32 * 128), bd,
                                    pl == 2 ? id_s : id_u, ks > 0);
                }
                ptx::mma_commit(&empty[stage]);
                ptx::mma_commit(&tfull[ab]);
                if (++stage == C::STAGES) stage = 0, phase ^= 1;
            }
        }
    } else {
        const int et = threadIdx.x - 64;                 // 0 .. 32 * kOmEpiWarps - 1
        const int q = warp & 3, pp = (warp - 2) >> 2;    // lane quarter = tile of the unit, output part
        const int cnt = min(C::PART, C::MM - pp * C::PART);
        const double sa = qpp->sa, rq = o.requant;
        // staged words per output channel: odd (conflict-free staging) for single columns, even
        // for the 8-byte pair loads
        constexpr int OCSK = (C::M % 2 == 0 && MK == 16) ? C::M * C::ROW + 2 : C::M * C::ROW + 1;
        for (int i = et; i < g.OC; i += 32 * kOmEpiWarps) {
            const double sc = (sa * sf[i]) / double(T::DEN * T::DEN);
            s_scale[i] = sc;
            s_scalef[i] = float(sc);
        }
        const int WO = g.WO, HO = g.HO, plane = HO * WO;
        const int tiles_img = g.th * g.tw;
        // column pairs (8-byte shared loads, 2-byte stores) for int8-only outputs of the even-M
        // variants; single columns otherwise (measured: pairs help the int8 layers of configs
        // 3-4, not the int32 outputs of config 5)
        constexpr int PW = (C::M % 2 == 0 && MK == 16) ? 2 : 1;
        constexpr int CPR = C::ROW / PW;                 // column items per staged row
        constexpr int NG = (32 * kOmEpiWarps) / CPR;     // channel groups of the store phase
        const int x_col = PW * (et % CPR), x_grp = et / CPR, x_tt = x_col / C::M, x_t2 = x_col % C::M;
        int rofs[C::M];  // row offsets t1 * WO
#pragma unroll
        for (int t1 = 0; t1 < C::M; ++t1) rofs[t1] = t1 * WO;
        int i = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
            const int ob = u % n_ob, tg = u / n_ob, ab = i & 1;
            int* sy = s_y + ab * (C::Y_BYTES / 4);
            TileInfo* st = s_tile + ab * kUnitTiles;
            ptx::mbar_wait_sleep(&tfull[ab], (i >> 1) & 1);
            ptx::tc_fence_after();
            uint32_t y[C::NP];
            {
                int32_t d0[C::NP], d1[C::NP], d2[C::NP];
                const uint32_t base = tmem + (uint32_t(q * 32) << 16) + uint32_t(ab * 3 * C::N + pp * C::NP);
#pragma unroll
                for (int c = 0; c < C::NP; c += 8) {
                    ptx::tmem_ld8(base + c, d0 + c);
                    ptx::tmem_ld8(base + C::N + c, d1 + c);
                    ptx::tmem_ld8(base + 2 * C::N + c, d2 + c);
                }
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < C::NP; ++c)  // exact mod 2^32: |y| < 2^31
                    y[c] = uint32_t(d0[c]) + (uint32_t(d1[c]) << 8) + (uint32_t(d2[c]) << 16);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[ab]);
            // staging into buffer ab: its previous readers (unit i - 2) finished before the
            // barrier of unit i - 1, which every thread has passed
            if (et < kUnitTiles) {
                const int t = tg * kUnitTiles + et;
                TileInfo ti{0, 0, 0};
                if (t < g.T) {
                    const int b = t / tiles_img, r = t - b * tiles_img, tr = r / g.tw, tc = r - tr * g.tw;
                    ti.base = ((long long)(b) * g.OC + ob * kUnitOc) * plane + (long long)(tr * C::M) * WO + tc * C::M;
                    ti.rows = min(C::M, HO - tr * C::M);
                    ti.cols = min(C::M, WO - tc * C::M);
                }
                st[et] = ti;
            }
            int* yr = sy + lane * OCSK;
#pragma unroll
            for (int c = 0; c < C::NP; ++c)
                if (c < cnt) {
                    const int oo = pp * C::PART + c, t1 = oo / C::M, t2 = oo % C::M;
                    yr[t1 * C::ROW + q * C::M + t2] = int(y[c]);
                }
            named_bar_epi();
            // stores: thread et keeps a column pair (x, x + 1) = PW (et % (ROW / PW)) of the unit's
            // staged rows (tile x / M, columns t2 (+1) of that tile; pairs for the even M of the
            // 6x6 / 4x4 variants) and walks output channels oc = et / (ROW / PW), + NG, ..., all
            // M rows each (predicated per row); consecutive threads write consecutive columns
            if (et < NG * CPR) {
                const TileInfo ti = st[x_tt];
                const int noc = min(kUnitOc, g.OC - ob * kUnitOc);
                const bool v0 = x_t2 < ti.cols, v1 = PW == 2 && x_t2 + 1 < ti.cols;
                const bool pair = v1 && (WO % 2 == 0);  // even element offsets: 2 / 8-byte stores
                if (v0) {
                    for (int oc = x_grp; oc < noc; oc += NG) {
                        const int ocg = ob * kUnitOc + oc;
                        const long long e0 = ti.base + x_t2 + (long long)oc * plane;
                        const int* ys = sy + oc * OCSK + x_col;
                        double sc = 0.0;
                        float scf = 0.f;
                        if ((MK ? (MK & 24) : (o.f64 || o.i8)) != 0) sc = s_scale[ocg];
                        if ((MK ? (MK & 4) : (o.f32 != nullptr)) != 0) scf = s_scalef[ocg];
                        int ya[C::M], yb[C::M];
#pragma unroll
                        for (int t1 = 0; t1 < C::M; ++t1) {
                            if constexpr (PW == 2) {
                                const int2 w = *reinterpret_cast<const int2*>(ys + t1 * C::ROW);
                                ya[t1] = w.x, yb[t1] = w.y;
                            } else {
                                ya[t1] = ys[t1 * C::ROW], yb[t1] = 0;
                            }
                        }
#pragma unroll
                        for (int t1 = 0; t1 < C::M; ++t1) {
                            const bool ok = t1 < ti.rows;
                            const long long e = e0 + rofs[t1];
                            if ((MK ? (MK & 1) : (o.y32 != nullptr))) {
                                if (ok && pair) *reinterpret_cast<int2*>(o.y32 + e) = make_int2(ya[t1], yb[t1]);
                                else {
                                    if (ok) o.y32[e] = ya[t1];
                                    if (ok && v1) o.y32[e + 1] = yb[t1];
                                }
                            }
                            if ((MK ? (MK & 2) : (o.y64 != nullptr))) {
                                if (ok) o.y64[e] = ya[t1];
                                if (ok && v1) o.y64[e + 1] = yb[t1];
                            }
                            if ((MK ? (MK & 4) : (o.f32 != nullptr))) {
                                const float fa = __int2float_rn(ya[t1]) * scf, fb = __int2float_rn(yb[t1]) * scf;
                                if (ok && pair) *reinterpret_cast<float2*>(o.f32 + e) = make_float2(fa, fb);
                                else {
                                    if (ok) o.f32[e] = fa;
                                    if (ok && v1) o.f32[e + 1] = fb;
                                }
                            }
                            if ((MK ? (MK & 8) : (o.f64 != nullptr))) {
                                if (ok) o.f64[e] = double(ya[t1]) * sc;
                                if (ok && v1) o.f64[e + 1] = double(yb[t1]) * sc;
                            }
                            if ((MK ? (MK & 16) : (o.i8 != nullptr))) {
                                const int qa = requant_i8(double(ya[t1]) * sc * rq);
                                const int qb = requant_i8(double(yb[t1]) * sc * rq);
                                int8_t* d = o.i8 + e;
                                if (ok && pair) *reinterpret_cast<uint16_t*>(d) = uint16_t((qa & 0xff) | ((qb & 0xff) << 8));
                                else {
                                    if (ok) d[0] = int8_t(qa);
                                    if (ok && v1) d[1] = int8_t(qb);
                                }
                            }
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    tl_mark(kTlOutput, 2);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

template <int V, int MK>
cudaError_t om_launch(const void* P, const ConvGeom& g, const QuantParams* qp, const double* sf, const OutPtrs& o,
                      cudaStream_t st, bool pdl) {
    using C = Om<V>;
    auto kern = k_out_mma<V, MK>;
    static SmemOptIn opt_in;
    if (cudaError_t e = opt_in.ensure(kern, C::SMEM); e != cudaSuccess) return e;
    const int n_ob = g.OCpad / kUnitOc, n_tg = g.Tpad / kUnitTiles;
    const int n_tg_used = (g.T + kUnitTiles - 1) / kUnitTiles;
    const long units = long(n_ob) * n_tg_used;
    if (units > 0x7fffffffL) return cudaErrorInvalidConfiguration;
    long grid = std::min<long>(units, device_sm_count());
    if (const char* e = std::getenv("SFC_OUT_GRID")) {  // experiment knob: cap the persistent grid
        const long cap = std::atol(e);
        if (cap > 0 && cap < grid) grid = cap;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kOmThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CUtensorMap tm;
    if (!make_pu_map(&tm, const_cast<void*>(P), g, C::F, 1, C::F, false)) return cudaErrorInvalidValue;
    return cudaLaunchKernelEx(&cfg, kern, tm, g, qp, sf, o, n_ob, n_tg, int(units));
}
// the output sets of the BASELINE workloads get their own specialisation (no predicated-off
// conversions in the store loop); any other set reads the pointers at run time
template <int V>
cudaError_t om_by_mask(const void* P, const ConvGeom& g, const QuantParams* qp, const double* sf, const OutPtrs& o,
                       cudaStream_t st, bool pdl) {
    const int mask = (o.y32 ? 1 : 0) | (o.y64 ? 2 : 0) | (o.f32 ? 4 : 0) | (o.f64 ? 8 : 0) | (o.i8 ? 16 : 0);
    switch (mask) {
        case 16: return om_launch<V, 16>(P, g, qp, sf, o, st, pdl);
        case 1: return om_launch<V, 1>(P, g, qp, sf, o, st, pdl);
        case 5: return om_launch<V, 5>(P, g, qp, sf, o, st, pdl);
        case 4: return om_launch<V, 4>(P, g, qp, sf, o, st, pdl);
        default: return om_launch<V, 0>(P, g, qp, sf, o, st, pdl);
    }
}
}  // namespace

bool output_mma_supported(int variant, const ConvGeom& g, const OutPtrs& o) {
    return variant <= 2 && g.p24 == 2 && g.OC <= kOmMaxOc && g.row0 == 0 && !o.p_discard &&
           (o.y32 || o.y64 || o.f32 || o.f64 || o.i8);
}

cudaError_t launch_output_mma(int variant, const void* P, const ConvGeom& g, const QuantParams* qp, const double* sf,
                              const OutPtrs& o, cudaStream_t st, bool pdl) {
    if (!output_mma_supported(variant, g, o)) return cudaErrorNotSupported;
    switch (variant) {
        case 0: return om_by_mask<0>(P, g, qp, sf, o, st, pdl);
        case 1: return om_by_mask<1>(P, g, qp, sf, o, st, pdl);
        default: return om_by_mask<2>(P, g, qp, sf, o, st, pdl);
    }
}

}  // namespace sfcb200
