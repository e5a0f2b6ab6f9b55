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
// Grid (oc blocks, tile-column blocks, image rows): no runtime division to decode a block.
// Not persistent: a CTA needs ~62 KB, so two or three are resident per SM and hide each
// other's TMA / barrier latency (the persistent double-buffered form needed 115 KB and ran
// one CTA per SM at 25% warp occupancy on the 28x28 layers).  Shared strides are odd so
// lanes stepping oc hit distinct banks.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"
#include "devcache.hpp"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"
#include "transforms.cuh"

namespace sfcb200 {

// One value of a 24-bit P slice held as three byte planes (b0, b1 unsigned, b2 signed) of
// `pl` bytes each: P = b0 + 2^8 b1 + 2^16 b2.
__device__ __forceinline__ int p24_value(const uint8_t* __restrict__ sp, size_t pl, int e) {
    return (int(reinterpret_cast<const int8_t*>(sp + 2 * pl)[e]) << 16) | (int(sp[pl + e]) << 8) | int(sp[e]);
}

namespace {
constexpr int kOcc = 32;  // output channels per block (128-byte TMA rows)
constexpr int kOutThreads = 512;

template <int V>
__host__ __device__ constexpr int out_tb() {  // tile columns per block: ~40 KB of P per block
    return (40 * 1024) / (Tab<V>::F * kOcc * 4) < 1 ? 1 : (40 * 1024) / (Tab<V>::F * kOcc * 4);
}
static_assert(out_tb<0>() * Tab<0>::M <= 32 && out_tb<1>() * Tab<1>::M <= 32 && out_tb<2>() * Tab<2>::M <= 32 &&
                  out_tb<3>() * Tab<3>::M <= 32 && out_tb<4>() * Tab<4>::M <= 32,
              "a block's output row segment must fit the 32-entry magic table");

// MODE 3 (fp64 P, the float fast_conv2d path) and MODE 4 (fp64 P of the wide 9-16 bit
// quantized path) halve the tile columns per block: their P slice is twice as wide per element.
template <int V, int MODE>
__host__ __device__ constexpr int out_tbm() {
    return MODE >= 3 ? (out_tb<V>() / 2 < 1 ? 1 : out_tb<V>() / 2) : out_tb<V>();
}
template <int MODE>
using p_elem_t = typename std::conditional<MODE >= 3, double, int32_t>::type;

struct OutSmem {
    int qstride, ystride;
    size_t p_bytes, q_off, bar_off, bytes;
};

template <int V, int MODE, int TBX = 0>
__host__ __device__ inline OutSmem out_smem() {
    using T = Tab<V>;
    constexpr int TB = TBX ? TBX : out_tbm<V, MODE>();
    const size_t es = MODE == 0 ? 4 : 8;
    OutSmem s;
    s.qstride = kOcc | 1;
    s.ystride = (T::M * TB) | 1;
    const size_t y_bytes = size_t(T::M) * kOcc * s.ystride * es;
    s.p_bytes = size_t(T::F) * TB * kOcc * sizeof(p_elem_t<MODE>);
    if (y_bytes > s.p_bytes) s.p_bytes = y_bytes;  // s_y reuses the P slice
    s.q_off = (s.p_bytes + 127) & ~size_t(127);
    s.bar_off = (s.q_off + size_t(TB) * T::M * T::K * s.qstride * es + 15) & ~size_t(15);
    s.bytes = s.bar_off + 16;
    return s;
}
}  // namespace

// umulhi magics for the divisors 1..32 (ncol): t / d == umulhi(t, c_magic32[d]) for t < 2^16
__constant__ unsigned c_magic32[33] = {  // 0xffffffff / d + 1 (exact for t < 2^16; generated)
    0x00000000u, 0x00000000u, 0x80000000u, 0x55555556u, 0x40000000u, 0x33333334u, 0x2aaaaaabu, 0x24924925u,
    0x20000000u, 0x1c71c71du, 0x1999999au, 0x1745d175u, 0x15555556u, 0x13b13b14u, 0x12492493u, 0x11111112u,
    0x10000000u, 0x0f0f0f10u, 0x0e38e38fu, 0x0d79435fu, 0x0ccccccdu, 0x0c30c30du, 0x0ba2e8bbu, 0x0b21642du,
    0x0aaaaaabu, 0x0a3d70a4u, 0x09d89d8au, 0x097b425fu, 0x0924924au, 0x08d3dcb1u, 0x08888889u, 0x08421085u,
    0x08000000u};

// MODE 0: exact int32 y, 1: exact int64 y, 2: general QuantConfig (P dequantised per
// (oc, f) before the inverse transform, which then runs in fp64: quant.cpp:258-278),
// 3: fp64 P of the float path (fast_conv2d, conv.cpp:495-510), no dequantisation,
// 4: as 2 from an fp64 P (the exact-integer P of the 9-16 bit path, |P| < 2^53).
// TBX = 1 (small grids, config 2): one tile per block and 256 threads -- three times the
// blocks with a third of the per-thread chain, all resident in one wave.
template <int V, int MODE, bool P24 = false, int TBX = 0>
__global__ void __launch_bounds__(TBX ? 256 : kOutThreads, 2)
    k_output(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmP2, ConvGeom g,
             const QuantParams* __restrict__ qpp, const double* __restrict__ sf, OutPtrs o) {
    using T = Tab<V>;
    constexpr int K = T::K, M = T::M, TB = TBX ? TBX : out_tbm<V, MODE>();
    constexpr int NTH = TBX ? 256 : kOutThreads;
    constexpr bool Y64 = MODE == 1;
    using acc_t =
        typename std::conditional<MODE >= 2, double, typename std::conditional<Y64, long long, int>::type>::type;
    extern __shared__ __align__(128) uint8_t smem[];
    const OutSmem L = out_smem<V, MODE, TBX>();
    const p_elem_t<MODE>* sp = reinterpret_cast<const p_elem_t<MODE>*>(smem);  // [F][TB][kOcc]
    acc_t* s_y = reinterpret_cast<acc_t*>(smem);                 // [M][kOcc] rows of ystride (after stage A)
    acc_t* s_q = reinterpret_cast<acc_t*>(smem + L.q_off);       // [TB][M][K] rows of qstride
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    __shared__ double s_scale[kOcc];
    __shared__ float s_scalef[kOcc];

    // grid = (oc blocks, tile-column blocks, image rows b * th + ti of the chunk); P rows are
    // chunk-relative, the output position uses the absolute row g.row0 + row
    const int oc0 = blockIdx.x * kOcc, tc = blockIdx.y, row = blockIdx.z;
    tl_mark(kTlOutput, 0);
    // 24-bit P: the slice's byte planes b0, b1 (unsigned), b2 (signed), [F][TB][kOcc] each, at
    // 128-byte aligned offsets (TMA destinations)
    constexpr size_t kPl = (size_t(T::F) * TB * kOcc + 127) & ~size_t(127);
    const uint8_t* sp_b = smem;
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
        if constexpr (P24) {
            ptx::mbar_expect_tx(full, uint32_t(size_t(T::F) * TB * kOcc * 3));
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
                ptx::tma_load_3d(smem + pl * kPl, &tmP, full, pl * g.OCpad + oc0, row * g.tw + tc * TB, 0);
        } else {
            ptx::mbar_expect_tx(full, uint32_t(size_t(T::F) * TB * kOcc * sizeof(p_elem_t<MODE>)));
            ptx::tma_load_3d(smem, &tmP, full, oc0, row * g.tw + tc * TB, 0);
        }
    }
    const int arow = g.row0 + row;
    const int b = arow / g.th, ti = arow - b * g.th;  // per block: exact for any row count
    const int noc = min(kOcc, g.OC - oc0);
    const int ntb = min(TB, g.tw - tc * TB);
    if (threadIdx.x < kOcc && int(threadIdx.x) < noc) {
        const double sc = (qpp->sa * sf[oc0 + threadIdx.x]) / double(T::DEN * T::DEN);
        s_scale[threadIdx.x] = sc;
        s_scalef[threadIdx.x] = float(sc);
    }
    ptx::mbar_wait(full, 0);
    if (o.p_discard) {  // this block is the only reader of its rows' lines: drop them from L2 unwritten
        constexpr int kLines = int(kOcc * sizeof(p_elem_t<MODE>) / 128);
        const char* pb = static_cast<const char*>(o.p_discard);
        for (int i = threadIdx.x; i < T::F * ntb * kLines; i += NTH) {
            const int l = i % kLines, j = (i / kLines) % ntb, f = i / (kLines * ntb);
            const size_t e = (size_t(f) * g.Tpad + size_t(row) * g.tw + tc * TB + j) * g.OCpad + oc0;
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(pb + e * sizeof(p_elem_t<MODE>) + l * 128) : "memory");
        }
    }

    // stage A: items (tj, l, oc)
    for (int it = threadIdx.x; it < TB * K * kOcc; it += NTH) {
        const int oc = it % kOcc, l = (it / kOcc) % K, tj = it / (kOcc * K);
        if (tj >= ntb) continue;
        acc_t pk[K], qt[M];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int e = ((k * K + l) * TB + tj) * kOcc + oc;
            if constexpr (P24)
                pk[k] = acc_t(p24_value(sp_b, kPl, e));
            else
                pk[k] = sp[e];
        }
        if constexpr (MODE == 2 || MODE == 4) {  // pd[f] = double(pacc[f]) * sa(f) * fil(oc, f), left to right
            const int ocg = oc0 + oc < g.OC ? oc0 + oc : 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int f = k * K + l;
                pk[k] = __dmul_rn(__dmul_rn(pk[k], o.gen_act[o.gen_per_freq ? f : 0]), o.gen_fil[ocg * T::F + f]);
            }
        }
        inv1d<V>(pk, qt);
#pragma unroll
        for (int t1 = 0; t1 < M; ++t1) s_q[((tj * M + t1) * K + l) * L.qstride + oc] = qt[t1];
    }
    __syncthreads();

    // stage B: items (tj, t1, oc)
    for (int it = threadIdx.x; it < TB * M * kOcc; it += NTH) {
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

    // stage C: the block's output row segments r = (t1, oc), ncol columns each.  Thread t
    // keeps column c = t % ncol and walks rows r = t / ncol, + NTH / ncol, ...
    // (consecutive threads -> consecutive columns of a row: coalesced row segments); the
    // divisions by ncol <= 32 are multiply-highs from a constant table.  The set of
    // requested outputs is a compile-time mask (one specialisation per combination).
    const int WO = g.WO;
    const int col0 = tc * TB * M;
    const int ncol = min(ntb * M, WO - col0);           // <= TB * M <= 32
    const int hrows = min(M, g.HO - ti * M);
    const int plane = g.HO * WO;
    const size_t base0 = (size_t(b) * g.OC + oc0) * size_t(plane) + size_t(ti) * M * WO + col0;
    const unsigned nmag = c_magic32[ncol];
    const int r0 = ncol == 1 ? int(threadIdx.x) : int(__umulhi(threadIdx.x, nmag));
    const int c = int(threadIdx.x) - r0 * ncol;
    const int rstep = ncol == 1 ? NTH : int(__umulhi(unsigned(NTH), nmag));
    const double rq = o.requant;
    auto emit = [&](auto mask_c) {
        constexpr int MK = decltype(mask_c)::value;
        if (r0 >= rstep) return;
        for (int r = r0; r < M * kOcc; r += rstep) {
            const int oc = r % kOcc, t1 = r / kOcc;
            if (oc >= noc || t1 >= hrows) continue;
            const size_t x = base0 + unsigned(oc * plane + t1 * WO + c);
            const acc_t y = s_y[r * L.ystride + c];
            if constexpr (MODE < 2 && (MK & 1) != 0) o.y32[x] = int(y);
            if constexpr (MODE < 2 && (MK & 2) != 0) o.y64[x] = int64_t(y);
            if constexpr (MODE >= 2) {  // y = sum A A pd; out = y / N^2 (the reference's a = A / N)
                const double out = double(y) / double(T::DEN * T::DEN);
                if constexpr ((MK & 4) != 0) o.f32[x] = float(out);
                if constexpr ((MK & 8) != 0) o.f64[x] = out;
                if constexpr ((MK & 16) != 0) o.i8[x] = requant_i8(out * rq);
            } else {
                if constexpr ((MK & 4) != 0)
                    o.f32[x] = Y64 ? float(double(y) * s_scale[oc]) : __int2float_rn(int(y)) * s_scalef[oc];
                if constexpr ((MK & 8) != 0) o.f64[x] = double(y) * s_scale[oc];
                if constexpr ((MK & 16) != 0)
                    o.i8[x] = requant_i8(double(y) * s_scale[oc] * rq);
            }
        }
    };
    const int mask = (o.y32 ? 1 : 0) | (o.y64 ? 2 : 0) | (o.f32 ? 4 : 0) | (o.f64 ? 8 : 0) | (o.i8 ? 16 : 0);
    switch (mask) {
#define SFC_EMIT_CASE(m) \
    case m: emit(std::integral_constant<int, m>{}); break;
        SFC_EMIT_CASE(1) SFC_EMIT_CASE(2) SFC_EMIT_CASE(3) SFC_EMIT_CASE(4) SFC_EMIT_CASE(5) SFC_EMIT_CASE(6)
        SFC_EMIT_CASE(7) SFC_EMIT_CASE(8) SFC_EMIT_CASE(9) SFC_EMIT_CASE(10) SFC_EMIT_CASE(11) SFC_EMIT_CASE(12)
        SFC_EMIT_CASE(13) SFC_EMIT_CASE(14) SFC_EMIT_CASE(15) SFC_EMIT_CASE(16) SFC_EMIT_CASE(17) SFC_EMIT_CASE(18)
        SFC_EMIT_CASE(19) SFC_EMIT_CASE(20) SFC_EMIT_CASE(21) SFC_EMIT_CASE(22) SFC_EMIT_CASE(23) SFC_EMIT_CASE(24)
        SFC_EMIT_CASE(25) SFC_EMIT_CASE(26) SFC_EMIT_CASE(27) SFC_EMIT_CASE(28) SFC_EMIT_CASE(29) SFC_EMIT_CASE(30)
        SFC_EMIT_CASE(31)
#undef SFC_EMIT_CASE
        default: break;
    }
    __syncthreads();
    tl_mark(kTlOutput, 2);
}

// ---------------------------------------------------------------------------------------
// Persistent output transform for the exact integer modes of the 3x3 variants over the
// [F][Tpad][OCpad] P layout.  Blocks as k_output (oc block of 32, TB tile columns of one
// image tile row); one thread per (tile, oc) pair.  Per block: wait for the block's P slice
// (one 3-D TMA load), stage A reads the pair's K^2 values from the slice straight into
// registers (lanes = oc: conflict-free) and applies the first inverse pass; one barrier frees
// the slice and the NEXT block's TMA load is issued at once, so it lands while this block
// runs stage B (second inverse pass, y parked in shared memory) and stage C (coalesced
// row-segment stores).  The transforms never round-trip through shared memory.
// Stage C of the register output kernels: the block's row segments r = (t1, oc) of ncol
// columns from s_y (rows of ys), all requested outputs (compile-time mask MK).  Even WO:
// thread t keeps the column pair 2cp (cp = t % npair) and walks rows r = t / npair,
// + nt / npair, ... (8-byte loads and stores: output offsets are even); odd WO (or pairs
// off): single columns.
template <int MK, bool Y64, int M, class acc_t>
__device__ __forceinline__ void emit_rows(const acc_t* __restrict__ s_y, int ys, int nt, int noc, int hrows,
                                          size_t base0, int plane, int WO, int ncol, bool pairs,
                                          const double* __restrict__ scl, const float* __restrict__ sclf, double rq,
                                          const OutPtrs& o) {
    const int nit = pairs ? (ncol + 1) >> 1 : ncol;  // items per row
    const unsigned nmag = c_magic32[nit];
    const int r0 = nit == 1 ? int(threadIdx.x) : int(__umulhi(threadIdx.x, nmag));
    const int ci = int(threadIdx.x) - r0 * nit;
    const int rstep = nit == 1 ? nt : int(__umulhi(unsigned(nt), nmag));
    if (r0 >= rstep) return;
    if (pairs) {
        const int c = 2 * ci;
        const bool two = c + 1 < ncol;
        for (int r = r0; r < M * kOcc; r += rstep) {
            const int oc = r & (kOcc - 1), t1 = r >> 5;
            if (oc >= noc || t1 >= hrows) continue;
            const size_t x = base0 + unsigned(oc * plane + t1 * WO + c);
            acc_t y0, y1;
            if constexpr (Y64) {
                y0 = s_y[r * ys + c], y1 = s_y[r * ys + c + 1];
            } else {
                const int2 v = *reinterpret_cast<const int2*>(s_y + r * ys + c);
                y0 = v.x, y1 = v.y;
            }
            if (two) {
                if constexpr ((MK & 1) != 0) *reinterpret_cast<int2*>(o.y32 + x) = make_int2(int(y0), int(y1));
                if constexpr ((MK & 2) != 0) {
                    o.y64[x] = int64_t(y0);
                    o.y64[x + 1] = int64_t(y1);
                }
                if constexpr ((MK & 4) != 0) {
                    const float2 f = Y64 ? make_float2(float(double(y0) * scl[oc]), float(double(y1) * scl[oc]))
                                         : make_float2(__int2float_rn(int(y0)) * sclf[oc],
                                                       __int2float_rn(int(y1)) * sclf[oc]);
                    *reinterpret_cast<float2*>(o.f32 + x) = f;
                }
                if constexpr ((MK & 8) != 0) {
                    o.f64[x] = double(y0) * scl[oc];
                    o.f64[x + 1] = double(y1) * scl[oc];
                }
                if constexpr ((MK & 16) != 0) {
                    const int q0 = int(requant_i8(double(y0) * scl[oc] * rq));
                    const int q1 = int(requant_i8(double(y1) * scl[oc] * rq));
                    *reinterpret_cast<int16_t*>(o.i8 + x) = int16_t(q0 | (q1 << 8));
                }
            } else {
                if constexpr ((MK & 1) != 0) o.y32[x] = int(y0);
                if constexpr ((MK & 2) != 0) o.y64[x] = int64_t(y0);
                if constexpr ((MK & 4) != 0)
                    o.f32[x] = Y64 ? float(double(y0) * scl[oc]) : __int2float_rn(int(y0)) * sclf[oc];
                if constexpr ((MK & 8) != 0) o.f64[x] = double(y0) * scl[oc];
                if constexpr ((MK & 16) != 0) o.i8[x] = requant_i8(double(y0) * scl[oc] * rq);
            }
        }
    } else {
        const int c = ci;
        for (int r = r0; r < M * kOcc; r += rstep) {
            const int oc = r & (kOcc - 1), t1 = r >> 5;
            if (oc >= noc || t1 >= hrows) continue;
            const size_t x = base0 + unsigned(oc * plane + t1 * WO + c);
            const acc_t y = s_y[r * ys + c];
            if constexpr ((MK & 1) != 0) o.y32[x] = int(y);
            if constexpr ((MK & 2) != 0) o.y64[x] = int64_t(y);
            if constexpr ((MK & 4) != 0) o.f32[x] = Y64 ? float(double(y) * scl[oc]) : __int2float_rn(int(y)) * sclf[oc];
            if constexpr ((MK & 8) != 0) o.f64[x] = double(y) * scl[oc];
            if constexpr ((MK & 16) != 0) o.i8[x] = requant_i8(double(y) * scl[oc] * rq);
        }
    }
}

// Runtime output mask -> emit_rows<MK>.
template <bool Y64, int M, class acc_t>
__device__ __forceinline__ void emit_rows_any(int mask, const acc_t* __restrict__ s_y, int ys, int nt, int noc,
                                              int hrows, size_t base0, int plane, int WO, int ncol, bool pairs,
                                              const double* __restrict__ scl, const float* __restrict__ sclf,
                                              double rq, const OutPtrs& o) {
    switch (mask) {
#define SFC_EMIT_CASE(m)                                                                                      \
    case m:                                                                                                   \
        emit_rows<m, Y64, M>(s_y, ys, nt, noc, hrows, base0, plane, WO, ncol, pairs, scl, sclf, rq, o); \
        break;
        SFC_EMIT_CASE(1) SFC_EMIT_CASE(2) SFC_EMIT_CASE(3) SFC_EMIT_CASE(4) SFC_EMIT_CASE(5) SFC_EMIT_CASE(6)
        SFC_EMIT_CASE(7) SFC_EMIT_CASE(8) SFC_EMIT_CASE(9) SFC_EMIT_CASE(10) SFC_EMIT_CASE(11) SFC_EMIT_CASE(12)
        SFC_EMIT_CASE(13) SFC_EMIT_CASE(14) SFC_EMIT_CASE(15) SFC_EMIT_CASE(16) SFC_EMIT_CASE(17) SFC_EMIT_CASE(18)
        SFC_EMIT_CASE(19) SFC_EMIT_CASE(20) SFC_EMIT_CASE(21) SFC_EMIT_CASE(22) SFC_EMIT_CASE(23) SFC_EMIT_CASE(24)
        SFC_EMIT_CASE(25) SFC_EMIT_CASE(26) SFC_EMIT_CASE(27) SFC_EMIT_CASE(28) SFC_EMIT_CASE(29) SFC_EMIT_CASE(30)
        SFC_EMIT_CASE(31)
#undef SFC_EMIT_CASE
        default: break;
    }
}

// int8-only stage C (the small-channel kernel's VGG-16 layer 0 output): thread t keeps the
// column pair 2 (t % npair) and walks rows r = (t1, oc) = t / npair, + nt / npair, ...; two
// values per 8-byte shared load and 2-byte store (even WO).
template <int M>
__device__ __forceinline__ void emit_rows_i8(const int* __restrict__ s_y, int ys, int nt, int noc, int hrows,
                                             size_t base0, int plane, int WO, int ncol,
                                             const double* __restrict__ scl, double rq, int8_t* __restrict__ out) {
    const int npair = (ncol + 1) >> 1;
    const unsigned nmag = c_magic32[npair];
    const int r0 = npair == 1 ? int(threadIdx.x) : int(__umulhi(threadIdx.x, nmag));
    const int c = 2 * (int(threadIdx.x) - r0 * npair);
    const int rstep = npair == 1 ? nt : int(__umulhi(unsigned(nt), nmag));
    if (r0 >= rstep) return;
    const bool two = c + 1 < ncol, pair = two && (WO & 1) == 0;
    for (int r = r0; r < M * kOcc; r += rstep) {
        const int oc = r & (kOcc - 1), t1 = r >> 5;
        if (oc >= noc || t1 >= hrows) continue;
        const int2 v = *reinterpret_cast<const int2*>(s_y + r * ys + c);
        const double sc = scl[oc];
        int qa, qb;
        if (fabs(sc * rq) < 1.0) {  // |y sc rq| < 2^31: the conversions on the fp64 add pipe (common.cuh)
            qa = requant_i8_small(v.x, sc, rq), qb = requant_i8_small(v.y, sc, rq);
        } else {
            qa = requant_i8(double(v.x) * sc * rq), qb = requant_i8(double(v.y) * sc * rq);
        }
        int8_t* d = out + base0 + unsigned(oc * plane + t1 * WO + c);
        if (pair) {
            *reinterpret_cast<uint16_t*>(d) = uint16_t((qa & 0xff) | ((qb & 0xff) << 8));
        } else {
            d[0] = int8_t(qa);
            if (two) d[1] = int8_t(qb);
        }
    }
}

template <int V>
struct PersSmem {
    static constexpr int TB = out_tb<V>();
    static constexpr int YS = ((Tab<V>::M * TB + 1) & ~1) | 2;  // = 2 (mod 4): 8-byte aligned rows
    static constexpr size_t slice = size_t(Tab<V>::F) * TB * kOcc * 4;
    template <bool Y64>
    static constexpr size_t y_bytes() { return size_t(Tab<V>::M) * kOcc * YS * (Y64 ? 8 : 4); }
    template <bool Y64>
    static constexpr size_t bytes() { return ((slice + 127) & ~size_t(127)) + y_bytes<Y64>() + 16; }
};

template <int V, bool Y64, bool P24>
__global__ void __launch_bounds__(32 * out_tb<V>()) k_output_pers(const __grid_constant__ CUtensorMap tmP,
                                                                  const __grid_constant__ CUtensorMap tmP2, ConvGeom g,
                                                                  const QuantParams* __restrict__ qpp,
                                                                  const double* __restrict__ sf, OutPtrs o, int n_ob,
                                                                  int n_tc, int nblk) {
    using T = Tab<V>;
    using PS = PersSmem<V>;
    constexpr int K = T::K, M = T::M, TB = PS::TB, NT = 32 * TB, YS = PS::YS;
    using acc_t = typename std::conditional<Y64, long long, int>::type;
    extern __shared__ __align__(128) uint8_t smem[];
    const int32_t* sp = reinterpret_cast<const int32_t*>(smem);  // [F][TB][kOcc]
    acc_t* s_y = reinterpret_cast<acc_t*>(smem + ((PS::slice + 127) & ~size_t(127)));  // rows (t1, oc) of YS
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + ((PS::slice + 127) & ~size_t(127)) + PS::template y_bytes<Y64>());
    __shared__ double s_scale[kOcc];
    __shared__ float s_scalef[kOcc];
    const int lane = threadIdx.x & 31, tjl = threadIdx.x >> 5;
    tl_mark(kTlOutput, 0);
    // P24: byte planes b0, b1, b2 of [F][TB][kOcc] at 128-byte aligned offsets (TMA destinations)
    constexpr size_t kPl = (size_t(T::F) * TB * kOcc + 127) & ~size_t(127);
    const uint8_t* sp_b = smem;
    auto issue = [&](int blk) {  // thread 0: the block's P slice
        const int ob = blk % n_ob, r = blk / n_ob, tc = r % n_tc, row = r / n_tc;
        if constexpr (P24) {
            ptx::mbar_expect_tx(full, uint32_t(size_t(T::F) * TB * kOcc * 3));
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
                ptx::tma_load_3d(smem + pl * kPl, &tmP, full, pl * g.OCpad + ob * kOcc, row * g.tw + tc * TB, 0);
        } else {
            ptx::mbar_expect_tx(full, uint32_t(PS::slice));
            ptx::tma_load_3d(smem, &tmP, full, ob * kOcc, row * g.tw + tc * TB, 0);
        }
    };
    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tmP);
        ptx::mbar_init(full, 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    griddep_wait();  // P complete
    tl_mark(kTlOutput, 1);
    griddep_launch_dependents();
    if (threadIdx.x == 0 && int(blockIdx.x) < nblk) issue(blockIdx.x);
    const double sa = qpp->sa;
    const double rq = o.requant;
    const int WO = g.WO, plane = g.HO * WO;
    const int mask = (o.y32 ? 1 : 0) | (o.y64 ? 2 : 0) | (o.f32 ? 4 : 0) | (o.f64 ? 8 : 0) | (o.i8 ? 16 : 0);
    uint32_t phase = 0;
    for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int ob = blk % n_ob, rr = blk / n_ob, tc = rr % n_tc, row = rr / n_tc;
        const int oc0 = ob * kOcc;
        const int arow = g.row0 + row;
        const int b = arow / g.th, ti = arow - b * g.th;  // per block: exact for any row count
        const int noc = min(kOcc, g.OC - oc0);
        const int ntb = min(TB, g.tw - tc * TB);
        const bool act = tjl < ntb;
        ptx::mbar_wait(full, phase);
        phase ^= 1;
        // stage A: Q[k][t2] = sum_l P[k*K + l] A[l][t2], P straight from the slice
        acc_t q[K][M];
        if (act) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                acc_t pr[K], qt[M];
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    const int e = ((k * K + l) * TB + tjl) * kOcc + lane;
                    if constexpr (P24)
                        pr[l] = acc_t(p24_value(sp_b, kPl, e));
                    else
                        pr[l] = acc_t(sp[e]);
                }
                inv1d<V>(pr, qt);
#pragma unroll
                for (int t2 = 0; t2 < M; ++t2) q[k][t2] = qt[t2];
            }
        }
        __syncthreads();  // slice consumed; the previous block's stage C is done with s_y / s_scale
        if (threadIdx.x == 0 && blk + int(gridDim.x) < nblk) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async write
            issue(blk + gridDim.x);
        }
        if (threadIdx.x < kOcc && int(threadIdx.x) < noc) {
            const double sc = (sa * sf[oc0 + threadIdx.x]) / double(T::DEN * T::DEN);
            s_scale[threadIdx.x] = sc;
            s_scalef[threadIdx.x] = float(sc);
        }
        // stage B: y[t1][t2] = sum_k A[k][t1] Q[k][t2] -> s_y
        if (act) {
#pragma unroll
            for (int t2 = 0; t2 < M; ++t2) {
                acc_t qc[K], yt[M];
#pragma unroll
                for (int k = 0; k < K; ++k) qc[k] = q[k][t2];
                inv1d<V>(qc, yt);
#pragma unroll
                for (int t1 = 0; t1 < M; ++t1) s_y[(t1 * kOcc + lane) * YS + tjl * M + t2] = yt[t1];
            }
        }
        __syncthreads();
        // stage C: coalesced row segments (emit_rows)
        const int col0 = tc * TB * M;
        const int ncol = min(ntb * M, WO - col0);  // <= TB * M <= 32
        const int hrows = min(M, g.HO - ti * M);
        const size_t base0 = (size_t(b) * g.OC + oc0) * size_t(plane) + size_t(ti) * M * WO + col0;
        emit_rows_any<Y64, M>(mask, s_y, YS, NT, noc, hrows, base0, plane, WO, ncol, (WO & 1) == 0 && o.pairs, s_scale,
                              s_scalef, rq, o);
    }
    tl_mark(kTlOutput, 2);
}

// ---------------------------------------------------------------------------------------
// Layers with at most 4 input channels (VGG-16's first layer, Cin = 3): the per-frequency
// contraction has K <= 4, so the tensor-core GEMM would spend its time writing P (4 B per
// (frequency, tile, oc); 4.7 GB on VGG-16 layer 0) for three multiply-adds per value.
// Here the contraction is one dp4a per (frequency, tile, oc) -- vq as one int8x4 word per
// (frequency, tile) (compact [F][T][4], written by the quantizing transform), the block's
// uq words [F][32] in shared memory -- fused with both inverse passes in registers and the
// coalesced row-segment stores of k_output.  P is never materialised; y is the same exact
// int32 (the contraction is the same integer sum).
constexpr int kSmallTB = 4;

// Persistent over tile blocks: a CTA keeps one oc block (its uq words staged once) and walks
// blocks (tc, row) = blockIdx.y, + gridDim.y, ...; per block the TB tiles' vq words [F][TB]
// are staged in shared memory (16-byte runs of the compact layout), then each thread forms
// its K^2 products with dp4a from two broadcast-free shared loads.
template <int V>
__global__ void __launch_bounds__(32 * kSmallTB) k_output_smallc(const int32_t* __restrict__ vq4,
                                                                 const int8_t* __restrict__ uq, ConvGeom g,
                                                                 const QuantParams* __restrict__ qpp,
                                                                 const double* __restrict__ sf, OutPtrs o, int n_tc,
                                                                 int nblk) {
    using T = Tab<V>;
    constexpr int K = T::K, M = T::M, F = T::F, TB = kSmallTB, NT = 32 * TB;
    constexpr int YS = ((M * TB + 1) & ~1) | 2;  // = 2 (mod 4): 8-byte aligned rows for the paired stores
    __shared__ int s_u[F * kOcc];      // uq words of this CTA's 32 output channels
    __shared__ int s_v[F * TB];        // vq words of the block's tiles
    __shared__ int s_y[M * kOcc * YS];  // rows r = (t1, oc) of YS
    __shared__ double s_scale[kOcc];
    __shared__ float s_scalef[kOcc];
    const int oc0 = blockIdx.x * kOcc;
    const int lane = threadIdx.x & 31, tjl = threadIdx.x >> 5;
    tl_mark(kTlOutput, 0);
    for (int i = threadIdx.x; i < F * kOcc; i += NT) {  // the layer's filters: before the wait
        const int f = i >> 5, oc = i & (kOcc - 1);
        s_u[i] = oc0 + oc < g.OCpad ? *reinterpret_cast<const int*>(uq + (size_t(f) * g.OCpad + oc0 + oc) * g.Cpad)
                                    : 0;
    }
    const int noc = min(kOcc, g.OC - oc0);
    griddep_wait();  // vq and the activation scale complete
    tl_mark(kTlOutput, 1);
    griddep_launch_dependents();
    if (threadIdx.x < kOcc && int(threadIdx.x) < noc) {  // (the same fp32 / fp64 epilogue as k_output)
        const double sc = (qpp->sa * sf[oc0 + threadIdx.x]) / double(T::DEN * T::DEN);
        s_scale[threadIdx.x] = sc;
        s_scalef[threadIdx.x] = float(sc);
    }
    const int WO = g.WO, plane = g.HO * WO;
    const double rq = o.requant;
    const int mask = (o.y32 ? 1 : 0) | (o.y64 ? 2 : 0) | (o.f32 ? 4 : 0) | (o.f64 ? 8 : 0) | (o.i8 ? 16 : 0);
    for (int blk = blockIdx.y; blk < nblk; blk += gridDim.y) {
        const int tc = blk % n_tc, row = blk / n_tc;
        const int arow = g.row0 + row;
        const int b = arow / g.th, ti = arow - b * g.th;  // per block: exact for any row count
        const int ntb = min(TB, g.tw - tc * TB);
        const int t0 = row * g.tw + tc * TB;
        __syncthreads();  // the previous block is done with s_v and s_y
        {
            constexpr int kPer = (F * TB + NT - 1) / NT;  // every load in flight before the stores
            int v[kPer];
#pragma unroll
            for (int jj = 0; jj < kPer; ++jj) {
                const int i = int(threadIdx.x) + jj * NT, f = i / TB, j = i - f * TB;
                v[jj] = i < F * TB && j < ntb ? __ldg(vq4 + size_t(f) * g.T + t0 + j) : 0;
            }
#pragma unroll
            for (int jj = 0; jj < kPer; ++jj)
                if (int(threadIdx.x) + jj * NT < F * TB) s_v[threadIdx.x + jj * NT] = v[jj];
        }
        __syncthreads();
        if (tjl < ntb) {
            int q[K][M];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                int pr[K], qt[M];
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    const int f = k * K + l;
                    pr[l] = __dp4a(s_v[f * TB + tjl], s_u[f * kOcc + lane], 0);
                }
                inv1d<V>(pr, qt);
#pragma unroll
                for (int t2 = 0; t2 < M; ++t2) q[k][t2] = qt[t2];
            }
#pragma unroll
            for (int t2 = 0; t2 < M; ++t2) {
                int qc[K], yt[M];
#pragma unroll
                for (int k = 0; k < K; ++k) qc[k] = q[k][t2];
                inv1d<V>(qc, yt);
#pragma unroll
                for (int t1 = 0; t1 < M; ++t1) s_y[(t1 * kOcc + lane) * YS + tjl * M + t2] = yt[t1];
            }
        }
        __syncthreads();
        // stage C: coalesced row segments (emit_rows)
        const int col0 = tc * TB * M;
        const int ncol = min(ntb * M, WO - col0);
        const int hrows = min(M, g.HO - ti * M);
        const size_t base0 = (size_t(b) * g.OC + oc0) * size_t(plane) + size_t(ti) * M * WO + col0;
        if (mask == 16) {  // int8 only (configs 3-4)
            if (ntb == TB && hrows == M && ncol == TB * M && noc == kOcc && (WO & 1) == 0 && M % 2 == 0) {
                // whole block (TB full tiles x M rows x 32 channels): thread items (oc, column pair) walk
                // the M rows with the scale, the base pointer and the row stride hoisted -- no predicates
                constexpr int NP2 = TB * M / 2;  // column pairs per staged row
                for (int it = threadIdx.x; it < kOcc * NP2; it += NT) {
                    const int oc = it / NP2, c = 2 * (it - oc * NP2);
                    const double sc = s_scale[oc];
                    int8_t* d = o.i8 + base0 + unsigned(oc * plane + c);
                    const int* ys = s_y + oc * YS + c;
                    if (fabs(sc * rq) < 1.0) {
#pragma unroll
                        for (int t1 = 0; t1 < M; ++t1) {
                            const int2 v = *reinterpret_cast<const int2*>(ys + t1 * (kOcc * YS));
                            const int qa = requant_i8_small(v.x, sc, rq), qb = requant_i8_small(v.y, sc, rq);
                            *reinterpret_cast<uint16_t*>(d + t1 * WO) = uint16_t(__byte_perm(uint32_t(qa), uint32_t(qb), 0x0040));
                        }
                    } else {
#pragma unroll
                        for (int t1 = 0; t1 < M; ++t1) {
                            const int2 v = *reinterpret_cast<const int2*>(ys + t1 * (kOcc * YS));
                            const int qa = requant_i8(double(v.x) * sc * rq), qb = requant_i8(double(v.y) * sc * rq);
                            *reinterpret_cast<uint16_t*>(d + t1 * WO) = uint16_t((qa & 0xff) | ((qb & 0xff) << 8));
                        }
                    }
                }
                continue;
            }
            emit_rows_i8<M>(s_y, YS, NT, noc, hrows, base0, plane, WO, ncol, s_scale, rq, o.i8);
            continue;
        }
        emit_rows_any<false, M>(mask, s_y, YS, NT, noc, hrows, base0, plane, WO, ncol, (WO & 1) == 0 && !o.i8, s_scale,
                                s_scalef, rq, o);
    }
    tl_mark(kTlOutput, 2);
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    // process-wide driver entry point, resolved once (thread-safe static initialisation)
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        return PFN_cuTensorMapEncodeTiled_v12000(nullptr);
    }();
    return fn;
}

// The output kernels' P slice maps: int32 / fp64 (box kOcc x TB x F), or the byte rows of the
// 24-bit layout (3*OCpad bytes: planes b0 | b1 | b2; box kOcc x TB x F, loaded once per plane).
bool make_slice_maps(CUtensorMap* tm, CUtensorMap* tm2, const void* P, const ConvGeom& g, int F, int TB, bool f64) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint32_t estr[3] = {1, 1, 1};
    *tm2 = CUtensorMap{};
    if (g.p24) {
        const cuuint64_t rb = cuuint64_t(g.OCpad) * 3;
        cuuint64_t dims[3] = {rb, cuuint64_t(g.Tpad), cuuint64_t(F)};
        cuuint64_t strides[2] = {rb, rb * g.Tpad};
        cuuint32_t box[3] = {kOcc, cuuint32_t(TB), cuuint32_t(F)};
        return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(P), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    const cuuint64_t es = f64 ? 8 : 4;
    cuuint64_t dims[3] = {cuuint64_t(g.OCpad), cuuint64_t(g.Tpad), cuuint64_t(F)};
    cuuint64_t strides[2] = {cuuint64_t(g.OCpad) * es, cuuint64_t(g.OCpad) * g.Tpad * es};
    cuuint32_t box[3] = {kOcc, cuuint32_t(TB), cuuint32_t(F)};
    return fn(tm, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_INT32, 3, const_cast<void*>(P), dims,
              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int V, int MODE, int TBX = 0>
cudaError_t out_launch(const void* P, const ConvGeom& g, const QuantParams* qp, const double* sf, const OutPtrs& o,
                       cudaStream_t st, bool pdl) {
    constexpr int TB = TBX ? TBX : out_tbm<V, MODE>();
    if constexpr (TBX == 0 && MODE <= 1) {  // small grids: one-tile blocks (fit one wave)
        const char* e = std::getenv("SFC_OUT_SMALL");
        const long nblk = long((g.OC + kOcc - 1) / kOcc) * ((g.tw + TB - 1) / TB) * g.nrows;
        const long nblk1 = long((g.OC + kOcc - 1) / kOcc) * g.tw * g.nrows;
        if (!(e && e[0] == '0') && !o.p_discard && nblk < 3L * 148 && nblk1 <= 8L * 148)
            return out_launch<V, MODE, 1>(P, g, qp, sf, o, st, pdl);
    }
    if (g.p24 && MODE > 1) return cudaErrorInvalidValue;
    CUtensorMap tm, tm2;
    if (!make_slice_maps(&tm, &tm2, P, g, Tab<V>::F, TB, MODE >= 3)) return cudaErrorInvalidValue;
    const size_t smem = out_smem<V, MODE, TBX>().bytes;
    auto kern = k_output<V, MODE, false, TBX>;
    if constexpr (MODE <= 1) {
        if (g.p24) kern = k_output<V, MODE, true, TBX>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const long rows = g.nrows;
    if (rows > 65535 || (g.tw + TB - 1) / TB > 65535) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((g.OC + kOcc - 1) / kOcc), unsigned((g.tw + TB - 1) / TB), unsigned(rows));
    cfg.blockDim = dim3(TBX ? 256 : kOutThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, tm, tm2, g, qp, sf, o);
}

int sm_count_out() { return device_sm_count(); }

template <int V, bool Y64>
cudaError_t out_pers_launch(const void* P, const ConvGeom& g, const QuantParams* qp, const double* sf,
                            const OutPtrs& o, cudaStream_t st, bool pdl) {
    using PS = PersSmem<V>;
    CUtensorMap tm, tm2;
    if (!make_slice_maps(&tm, &tm2, P, g, Tab<V>::F, PS::TB, false)) return cudaErrorInvalidValue;
    constexpr size_t smem = PS::template bytes<Y64>();
    auto kern = g.p24 ? k_output_pers<V, Y64, true> : k_output_pers<V, Y64, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const int n_ob = (g.OC + kOcc - 1) / kOcc, n_tc = (g.tw + PS::TB - 1) / PS::TB;
    const long nblk = long(n_ob) * n_tc * g.nrows;
    if (nblk > 0x7fffffffL) return cudaErrorInvalidConfiguration;
    int per_sm = int((220 * 1024) / (smem + 1024));
    per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
    const long grid = std::min<long>(nblk, long(sm_count_out()) * per_sm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(32 * PS::TB);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr2[1];
    attr2[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr2[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr2;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, tm, tm2, g, qp, sf, o, n_ob, n_tc, int(nblk));
}

bool out_pers_wanted(int variant, int mode, const ConvGeom& g, const OutPtrs& o) {
    // Measured (24-bit P): faster on every ResNet-18 / VGG-16 layer with int8 requant outputs
    // (VGG-16 11.37 -> 10.57 ms, ResNet-18 1.021 -> 0.999 ms) and on 512-channel int32 / fp32
    // layers (config 5); slower for wide int32 outputs on narrower layers (VGG-16 layer 1 y32
    // 1.49 vs 1.22 ms), which keep the one-block kernel.
    const char* fe = std::getenv("SFC_OUT_PERS");  // "0": never, "1": force (A/B knob)
    if (variant > 2 || mode > 1 || o.p_discard) return false;
    if (fe && fe[0] == '1') return true;
    const bool wide_out = o.y32 || o.y64 || o.f32 || o.f64;
    if (wide_out && g.OC < 512) return false;
    // small layers (config 2: 320 blocks) keep the 512-thread one-block CTAs: a persistent CTA
    // of 64-192 threads has the longer per-block latency chain
    const int tb = variant == 0 ? out_tb<0>() : variant == 1 ? out_tb<1>() : out_tb<2>();
    const long nblk = long((g.OC + kOcc - 1) / kOcc) * ((g.tw + tb - 1) / tb) * g.nrows;
    if (nblk < 8L * sm_count_out()) return false;
    return !fe || fe[0] != '0';
}

template <int V>
cudaError_t out_by_width(int mode, const void* P, const ConvGeom& g, const QuantParams* qp, const double* sf,
                         const OutPtrs& o, cudaStream_t st, bool pdl) {
    if (g.p24 == 2) {  // unit-major P: only the tensor-core output transform reads it
        if (mode != 0) return cudaErrorInvalidValue;
        return launch_output_mma(V, P, g, qp, sf, o, st, pdl);
    }
    if constexpr (V <= 2) {
        if (out_pers_wanted(V, mode, g, o)) {
            OutPtrs op = o;
            static const char* pe = std::getenv("SFC_OUT_PAIRS");  // "0": single columns (A/B knob)
            op.pairs = !(pe && pe[0] == '0');  // (config 5 0.110 vs 0.114 ms single columns)
            return mode == 0 ? out_pers_launch<V, false>(P, g, qp, sf, op, st, pdl)
                             : out_pers_launch<V, true>(P, g, qp, sf, op, st, pdl);
        }
    }
    return mode == 0 ? out_launch<V, 0>(P, g, qp, sf, o, st, pdl)
         : mode == 1 ? out_launch<V, 1>(P, g, qp, sf, o, st, pdl)
         : mode == 2 ? out_launch<V, 2>(P, g, qp, sf, o, st, pdl)
         : mode == 3 ? out_launch<V, 3>(P, g, qp, sf, o, st, pdl)
                     : out_launch<V, 4>(P, g, qp, sf, o, st, pdl);
}
}  // namespace

cudaError_t launch_output(int variant, int mode, const void* P, const ConvGeom& g, const QuantParams* qp,
                          const double* sf, const OutPtrs& o, cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return out_by_width<0>(mode, P, g, qp, sf, o, st, pdl);
        case 1: return out_by_width<1>(mode, P, g, qp, sf, o, st, pdl);
        case 2: return out_by_width<2>(mode, P, g, qp, sf, o, st, pdl);
        case 3: return out_by_width<3>(mode, P, g, qp, sf, o, st, pdl);
        default: return out_by_width<4>(mode, P, g, qp, sf, o, st, pdl);
    }
}

cudaError_t launch_output_smallc(int variant, const int8_t* vq4, const int8_t* uq, const ConvGeom& g,
                                 const QuantParams* qp, const double* sf, const OutPtrs& o, cudaStream_t st, bool pdl) {
    const int n_ob = (g.OC + kOcc - 1) / kOcc, n_tc = (g.tw + kSmallTB - 1) / kSmallTB;
    const long nblk = long(n_tc) * g.nrows;
    if (nblk > 0x7fffffffL || n_ob > 65535 || g.Cpad % 4) return cudaErrorInvalidConfiguration;
    // ~6 CTAs of 4 warps per SM (shared memory ~34 KB each), split over the oc blocks
    const long want = (long(sm_count_out()) * 6 + n_ob - 1) / n_ob;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(n_ob), unsigned(std::min<long>(std::min<long>(nblk, want), 65535)));
    cfg.blockDim = dim3(32 * kSmallTB);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    const int32_t* v = reinterpret_cast<const int32_t*>(vq4);
    switch (variant) {
        case 0: return cudaLaunchKernelEx(&cfg, k_output_smallc<0>, v, uq, g, qp, sf, o, n_tc, int(nblk));
        case 1: return cudaLaunchKernelEx(&cfg, k_output_smallc<1>, v, uq, g, qp, sf, o, n_tc, int(nblk));
        case 2: return cudaLaunchKernelEx(&cfg, k_output_smallc<2>, v, uq, g, qp, sf, o, n_tc, int(nblk));
        default: return cudaErrorInvalidValue;
    }
}

SFC_TL_UNIT_READER(tl_read_out)

cudaError_t launch_output(int variant, bool y64, const int32_t* P, const ConvGeom& g, const QuantParams* qp,
                          const double* sf, const OutPtrs& o, cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return out_by_width<0>(y64, P, g, qp, sf, o, st, pdl);
        case 1: return out_by_width<1>(y64, P, g, qp, sf, o, st, pdl);
        case 2: return out_by_width<2>(y64, P, g, qp, sf, o, st, pdl);
        case 3: return out_by_width<3>(y64, P, g, qp, sf, o, st, pdl);
        default: return out_by_width<4>(y64, P, g, qp, sf, o, st, pdl);
    }
}

}  // namespace sfcb200
