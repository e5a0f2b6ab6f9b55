// Stage 4 of the quantized SFC conv: the per-frequency channel contraction
//   P[f][t][oc] = sum_ic vq[f][t][ic] * uq[f][oc][ic]            (quant.cpp:251-257)
// as int8 x int8 -> int32 GEMMs on the 5th-gen tensor cores (tcgen05.mma kind::i8,
// accumulators in TMEM), operands staged by TMA with 128B/64B swizzle.
//
// Persistent static schedule: CTA i processes work units u = i, i + grid, ...,
// unit -> (f, t-block, oc-block) with the oc-block fastest so concurrently resident
// CTAs share a frequency's A/B tiles in L2.  Warp roles: 0 = TMA producer,
// 1 = MMA issuer (one elected lane) and TMEM owner, 2..9 = epilogue
// (tcgen05.ld -> 128B-swizzled smem box -> TMA store), two epilogue warps per lane
// quarter; with QF, 10..17 = converters that quantize the kept int16 V straight into the
// A stage buffers.  TMEM accumulators are double-buffered so unit u+1's MMAs overlap
// unit u's epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "devcache.hpp"
#include "sfc_kernels.hpp"

#ifdef GM_TRACE  // experiment build: clock stamps of CTA 0's first units per role, printed at exit
#include <cstdio>
#define GM_STAMP(role, unit, k) do { if (blockIdx.x == 0 && (unit) < 32) s_trace[((role) * 32 + (unit)) * 4 + (k)] = clock64(); } while (0)
#else
#define GM_STAMP(role, unit, k) do { } while (0)
#endif

namespace sfcb200 {

namespace {
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3,
                                             int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}
__device__ __forceinline__ void bulk_store_128(void* dst, const void* src) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(reinterpret_cast<uint64_t>(dst)),
                 "r"(ptx::smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int kEpiWarps = 8;                 // two epilogue warps per TMEM lane quarter
constexpr int kConvWarps = 8;                // QF: activation-quantizing A producers
constexpr int kEpiBufs = 2;                  // TMA-store staging boxes per epilogue warp
constexpr int kEpiBoxBytes = 32 * 32 * 4;    // 32 rows x 32 int32 (one 128B-swizzle box)
template <bool QF>
constexpr int gemm_threads() { return 64 + 32 * kEpiWarps + (QF ? 32 * kConvWarps : 0); }
// TMEM accumulator buffers: the epilogue warps take every unit in turn, so their per-unit latency
// bounds the kernel; with more than two buffers the MMAs run ahead and the epilogue never waits
// for them (BN = 64: 4 x 64 columns, still two CTAs per SM; the TMA-staged-V kernel is alone on
// its SM and takes 512 columns at BN = 128).
template <int BN, int BK, int STAGES, bool QT>
constexpr int gemm_acc() {
    // (a CTA whose shared memory leaves room for a second one on the SM shares the 512 columns with it)
    const size_t smem = size_t(STAGES) * (128 + BN) * BK + (QT ? size_t(STAGES) * 128 * BK * 2 : 0) + 64 * 1024 + 1280;
    const int share = 2 * smem <= 227 * 1024 ? 256 : 512;
    return share / BN >= 4 ? 4 : (share / BN >= 2 ? share / BN : 2);
}

// Work unit -> (oc block, tile block, frequency): oc block fastest, so co-resident CTAs share
// a frequency's A tile in L2.
__device__ __forceinline__ void unit_of(int u, int n_ob, int n_tb, int& ob, int& tb, int& f) {
    ob = u % n_ob, tb = (u / n_ob) % n_tb, f = u / (n_ob * n_tb);
}
// Frequency before tile block (A/B knob SFC_GEMM_FMAJOR=1 with unit-major P; ob stays fastest,
// so concurrent CTAs still share the A tile).
__device__ __forceinline__ void unit_of(int u, int n_ob, int n_tb, int F, bool f_major, int& ob, int& tb, int& f) {
    if (!f_major) return unit_of(u, n_ob, n_tb, ob, tb, f);
    ob = u % n_ob, f = (u / n_ob) % F, tb = u / (n_ob * F);
}

// The same unit sequence u = u0, u0 + stride, ... as mixed-radix digits (d0 fastest: the oc block; d1, d2 =
// (tile block, f) or, f_major, (f, tile block)) advanced by addition with carries -- no division per unit.
struct UnitWalk3 {
    int d0, d1, d2, s0, s1, s2, r0, r1;
    bool fm;
    __device__ __forceinline__ UnitWalk3(int u0, int stride, int n_ob, int n_tb, int F, bool f_major) : fm(f_major) {
        r0 = n_ob, r1 = f_major ? F : n_tb;
        d0 = u0 % r0, d1 = (u0 / r0) % r1, d2 = u0 / (r0 * r1);
        s0 = stride % r0, s1 = (stride / r0) % r1, s2 = stride / (r0 * r1);
    }
    __device__ __forceinline__ void get(int& ob, int& tb, int& f) const {
        ob = d0;
        if (fm) f = d1, tb = d2;
        else tb = d1, f = d2;
    }
    __device__ __forceinline__ void next() {
        d0 += s0;
        int c = 0;
        if (d0 >= r0) d0 -= r0, c = 1;
        d1 += s1 + c;
        c = 0;
        if (d1 >= r1) d1 -= r1, c = 1;
        d2 += s2 + c;
    }
};

// Byte planes 0..2 of four int32 values (a, b, c, d): p_j = [a.b_j, b.b_j, c.b_j, d.b_j] -- a
// 4x4 byte transpose restricted to three outputs, 7 byte permutes (instead of 9 per plane set).
__device__ __forceinline__ void byte_planes3(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t& p0,
                                             uint32_t& p1, uint32_t& p2) {
    const uint32_t lo_ab = __byte_perm(a, b, 0x5140), lo_cd = __byte_perm(c, d, 0x5140);  // [x.b0 y.b0 x.b1 y.b1]
    const uint32_t hi_ab = __byte_perm(a, b, 0x6262), hi_cd = __byte_perm(c, d, 0x6262);  // [x.b2 y.b2 ..]
    p0 = __byte_perm(lo_ab, lo_cd, 0x5410);
    p1 = __byte_perm(lo_ab, lo_cd, 0x7632);
    p2 = __byte_perm(hi_ab, hi_cd, 0x5410);
}

// Quantize the four int16 values of two int16x2 words (lanes: low then high half) and pack
// the four int8 results into one word: sign-extended halves, two byte permutes to pack.
template <class Q>
__device__ __forceinline__ uint32_t pack_q4(uint32_t w0, uint32_t w1, Q&& quant) {
    const int a0 = int(int16_t(w0)), a1 = int(w0) >> 16, b0 = int(int16_t(w1)), b1 = int(w1) >> 16;
    const uint32_t lo = __byte_perm(uint32_t(quant(a0)), uint32_t(quant(a1)), 0x0040);
    const uint32_t hi = __byte_perm(uint32_t(quant(b0)), uint32_t(quant(b1)), 0x0040);
    return __byte_perm(lo, hi, 0x5410);
}

// Quantizer parameters for a subset of warps (no CTA-wide barrier): table or warp derivation.
__device__ __forceinline__ QuantParams qparams_warp(int vmax, int bits, const QuantParams* __restrict__ tab) {
    if (tab && vmax >= 0 && vmax <= kQpTableMax && bits >= 2 && bits <= 8)
        return tab[(bits - 2) * (kQpTableMax + 1) + vmax];
    return derive_qparams_warp(vmax, bits);
}
}  // namespace

// QF = false: A = vq [F][Tpad][Cpad] int8 via TMA.  QF = true: A is produced by kConvWarps
// converter warps from the kept int16 V: each thread owns 16-channel chunks of A rows,
// quantizes them and stores the 16 bytes at the chunk's swizzled position (128B swizzle:
// chunk j of row r at j ^ (r & 7); 64B swizzle: j ^ ((r >> 1) & 3)), i.e. exactly the
// layout the TMA load would produce.  QT = false: the converters load their chunks from
// global memory into registers (double-buffered); QT = true: the producer TMA-loads the
// stage's V tile (128 rows x BK channels of int16, rows >= T and channels >= C zero-filled
// by the tensor map) into a shared V stage next to A and B, and the converters read it
// from there -- far more bytes in flight per SM than register staging allows.
template <int BN, int BK, int STAGES, bool QF, bool QT = false>
__global__ void __launch_bounds__(gemm_threads<QF>(), 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmP2,
           const __grid_constant__ CUtensorMap tmP3, int n_tb, int n_ob, int F, int nk, ConvGeom g, QFuse qf,
           uint8_t* __restrict__ p_raw) {
    static_assert(!QT || QF, "the TMA-staged V feeds the converters");
    constexpr int kAcc = gemm_acc<BN, BK, STAGES, QT>();  // TMEM accumulator buffers
    constexpr int kTmemCols = kAcc * BN <= 128 ? 128 : (kAcc * BN <= 256 ? 256 : 512);
    constexpr uint32_t kStageBytes = (kRowsPerTile + BN) * BK;
    constexpr uint32_t kVStageBytes = kRowsPerTile * BK * 2;
    constexpr int kHalf = BN / 2;                     // columns per epilogue warp (two warps per lane quarter)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = sA + STAGES * kRowsPerTile * BK;
    uint8_t* sV = sB + STAGES * BN * BK;              // QT: [STAGES][128 rows][BK] int16
    uint8_t* sE = sV + (QT ? STAGES * kVStageBytes : 0);  // [8 warps][kEpiBufs][32 rows x 128 B], 128B-swizzled
    uint64_t* full = reinterpret_cast<uint64_t*>(sE + kEpiWarps * kEpiBufs * kEpiBoxBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + kAcc;
    uint64_t* vfull = tempty + kAcc;                  // QT: V stage landed
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(vfull + (QT ? STAGES : 0));
#ifdef GM_TRACE
    long long* s_trace = reinterpret_cast<long long*>(tmem_holder + 2);
    int tu = 0;
#endif

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = F * n_tb * n_ob;
    tl_mark(kTlGemm, 0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], QF ? 1 + kConvWarps : 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < kAcc; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], kEpiWarps);
        }
        if (QT)
            for (int s2 = 0; s2 < STAGES; ++s2) ptx::mbar_init(&vfull[s2], 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        if (!QF || QT) ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        ptx::tma_prefetch(&tmP);
        if (g.p24 >= 2) ptx::tma_prefetch(&tmP2), ptx::tma_prefetch(&tmP3);
    }
    if (warp == 1) ptx::tmem_alloc(tmem_holder, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    griddep_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            // QF: B (the layer's filters) does not depend on the predecessor; the converters wait.
            if (!QF || QT) griddep_wait();  // vq / V written by the activation kernel
            tl_mark(kTlGemm, 1);
            int stage = 0;
            uint32_t phase = 0;
            UnitWalk3 uw(blockIdx.x, gridDim.x, n_ob, n_tb, F, g.p24 == 2);
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int ob, tb, f;
                uw.get(ob, tb, f);
                uw.next();
                for (int kc = 0; kc < nk; ++kc) {
                    ptx::mbar_wait_sleep<100>(&empty[stage], phase ^ 1);
                    GM_STAMP(0, tu, 0);
                    if (QF) {
                        ptx::mbar_expect_tx(&full[stage], uint32_t(BN * BK));
                        if (QT) {
                            ptx::mbar_expect_tx(&vfull[stage], kVStageBytes);
                            ptx::tma_load_3d(sV + stage * kVStageBytes, &tmA, &vfull[stage], kc * BK,
                                             tb * kRowsPerTile, f);
                        }
                    } else {
                        ptx::mbar_expect_tx(&full[stage], kStageBytes);
                        ptx::tma_load_3d(sA + stage * kRowsPerTile * BK, &tmA, &full[stage], kc * BK, tb * kRowsPerTile, f);
                    }
                    ptx::tma_load_3d(sB + stage * BN * BK, &tmB, &full[stage], kc * BK, ob * BN, f);
                    GM_STAMP(0, tu, 1);
                    if (++stage == STAGES) stage = 0, phase ^= 1;
                }
#ifdef GM_TRACE
                ++tu;
#endif
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_i8(kRowsPerTile, BN);
            int stage = 0;
            uint32_t phase = 0;
            int i = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
                const int ab = i % kAcc;
                ptx::mbar_wait(&tempty[ab], ((i / kAcc) & 1) ^ 1);
                GM_STAMP(1, i, 0);
                ptx::tc_fence_after();
                const uint32_t d = tmem + uint32_t(ab * BN);
                for (int kc = 0; kc < nk; ++kc) {
                    ptx::mbar_wait(&full[stage], phase);
                    GM_STAMP(1, i, 1);
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
                GM_STAMP(1, i, 2);
            }
        }
    } else if (warp < 2 + kEpiWarps) {
        // Epilogue: warp e = warp - 2 owns TMEM lane quarter (warp & 3) and column half e / 4.
        const int q = warp & 3, half = (warp - 2) >> 2;
        uint8_t* myE = sE + (warp - 2) * kEpiBufs * kEpiBoxBytes;
        int buf = 0;
        int i = 0;
        UnitWalk3 uw(blockIdx.x, gridDim.x, n_ob, n_tb, F, g.p24 == 2);
        int ab = 0;
        uint32_t aphase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
            int ob, tb, f;
            uw.get(ob, tb, f);
            uw.next();
            ptx::mbar_wait_sleep<100>(&tfull[ab], aphase);
            if (warp == 2 && lane == 0) GM_STAMP(2, i, 0);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = half * kHalf; c < (half + 1) * kHalf; c += 32) {
                int32_t r[32];
                ptx::tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(ab * BN + c), r);
                ptx::tmem_wait_ld();
                if (warp == 2 && lane == 0) GM_STAMP(2, i, 1);
                if (lane == 0) bulk_wait_read<kEpiBufs - 1>();  // this buffer's previous store has read smem
                __syncwarp();
                if (warp == 2 && lane == 0) GM_STAMP(2, i, 2);
                uint8_t* box = myE + buf * kEpiBoxBytes;
                uint32_t p2rows = 0;
                if (g.p24 >= 2) {
                    // unit-major 24-bit P (sfc_kernels.hpp pu_offset): this thread's tile t and 32
                    // channels are one 32-byte piece of row f of each byte plane of unit
                    // (oc block, t / 4), chunks 2 (t & 3) and 2 (t & 3) + 1 swizzled with f & 7;
                    // the warp's 8 units x 128 B rows per plane are staged as [8][128 B] and
                    // stored with one TMA box per plane (tmP2: the 5-D unit-major map)
                    // (the staging box is 128B-swizzled by the store map: row r = lane / 4 of the box
                    // holds global chunk c at c ^ r -- conflict-free 16-byte stores)
                    const int sw = (f & 7) ^ (lane >> 2), c0 = 2 * (lane & 3);
                    uint8_t* rb = box + (lane >> 2) * 128;
                    uint32_t wv[3][8];
                    if (g.p2s) {  // sparse plane 2: P' = P + 2^15 keeps 16-bit values in planes 0 and 1
#pragma unroll
                        for (int j = 0; j < 32; ++j) r[j] += 32768;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        byte_planes3(uint32_t(r[4 * j]), uint32_t(r[4 * j + 1]), uint32_t(r[4 * j + 2]),
                                     uint32_t(r[4 * j + 3]), wv[0][j], wv[1][j], wv[2][j]);
                    // rows of plane 2 to store: all (dense), or the units (4 lanes each) holding a
                    // value outside 16 bits
                    p2rows = 0xffffffffu;
                    if (g.p2s)
                        p2rows = __ballot_sync(0xffffffffu, (wv[2][0] | wv[2][1] | wv[2][2] | wv[2][3] | wv[2][4] |
                                                             wv[2][5] | wv[2][6] | wv[2][7]) != 0);
                    p2rows = (p2rows | (p2rows >> 1) | (p2rows >> 2) | (p2rows >> 3)) & 0x11111111u;  // bit 4u: unit u
                    // all eight units: the swizzled box and one TMA store; some: rows in their
                    // global chunk order (c ^ (f & 7)) for one 128-byte bulk store each
                    const int sw2 = p2rows == 0x11111111u ? sw : (f & 7);
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl) {
                        if (pl == 2 && p2rows == 0) break;
                        const int s2 = pl == 2 ? sw2 : sw;
                        *reinterpret_cast<uint4*>(rb + pl * 1024 + ((c0 ^ s2) << 4)) =
                            make_uint4(wv[pl][0], wv[pl][1], wv[pl][2], wv[pl][3]);
                        *reinterpret_cast<uint4*>(rb + pl * 1024 + (((c0 + 1) ^ s2) << 4)) =
                            make_uint4(wv[pl][4], wv[pl][5], wv[pl][6], wv[pl][7]);
                    }
                } else if (g.p24) {
                    // 24-bit P as three byte planes (b0, b1 unsigned, b2 signed: P = b0 + 2^8 b1 +
                    // 2^16 b2): row `lane` of three 32 x 32 B boxes (32B swizzle: chunk j at
                    // j ^ ((lane >> 2) & 1)); the byte planes are the int8 operands of the
                    // tensor-core output transform (out_mma.cu)
                    uint8_t* rb = box + lane * 32;
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl) {
                        const uint32_t sel = pl == 0 ? 0x0040u : (pl == 1 ? 0x0051u : 0x0062u);
                        uint32_t wv[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            wv[j] = __byte_perm(__byte_perm(uint32_t(r[4 * j]), uint32_t(r[4 * j + 1]), sel),
                                                __byte_perm(uint32_t(r[4 * j + 2]), uint32_t(r[4 * j + 3]), sel), 0x5410);
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            *reinterpret_cast<uint4*>(rb + pl * 1024 + ((j ^ ((lane >> 2) & 1)) << 4)) =
                                make_uint4(wv[4 * j], wv[4 * j + 1], wv[4 * j + 2], wv[4 * j + 3]);
                    }
                } else {
                    // row `lane` of a 32 x 32 int32 box, 16-byte chunk j stored at j ^ (lane & 7) (128B swizzle)
                    uint8_t* row = box + lane * 128;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<int4*>(row + ((j ^ (lane & 7)) << 4)) =
                            make_int4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
                }
                fence_async_smem();
                __syncwarp();
                if (g.p24 >= 2 && g.p2s && (lane & 3) == 0) {
                    // one flag byte per (unit, f): [oc block][tile group / 8][F][8]; lane 4 uu owns unit uu
                    const int t0u = (tb * kRowsPerTile + q * 32) / kUnitTiles, o0u = (ob * BN + c) / kUnitOc;
                    p_raw[p2_flags_offset(F, g.Tpad, g.OCpad) + p2_flag_index(o0u, t0u, f, g.Tpad, F) + (lane >> 2)] =
                        uint8_t((p2rows >> lane) & 1u);
                }
                if (lane == 0) {
                    const int t0 = tb * kRowsPerTile + q * 32, o0 = ob * BN + c;
                    if (g.p24 >= 2) {  // (row, f, plane, tile group, oc block)
                        const int t0u = (tb * kRowsPerTile + q * 32) / kUnitTiles, o0u = (ob * BN + c) / kUnitOc;
                        // planes 0 and 1 as one box (the staging is [plane][8 units][128 B]): a TMA
                        // store costs its issuing lane ~300 cycles
                        tma_store_5d(&tmP2, box, 0, t0u, f, 0, o0u);
                        if (p2rows == 0x11111111u) {
                            tma_store_5d(&tmP3, box + 2 * 1024, 0, t0u, f, 2, o0u);
                        } else if (p2rows) {
                            for (int uu = 0; uu < 8; ++uu)
                                if ((p2rows >> (4 * uu)) & 1u)
                                    bulk_store_128(p_raw + pu_offset(o0u, t0u + uu, 2, f, g.Tpad / kUnitTiles, F),
                                                   box + 2 * 1024 + uu * 128);
                        }
                    } else if (g.p24) {  // byte coordinates: plane j of a P row starts at j * OCpad
#pragma unroll
                        for (int pl = 0; pl < 3; ++pl) tma_store_3d(&tmP, box + pl * 1024, pl * g.OCpad + o0, t0, f);
                    } else {
                        tma_store_3d(&tmP, box, o0, t0, f);
                    }
                    bulk_commit();
                }
                buf = (buf + 1) % kEpiBufs;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[ab]);
            if (warp == 2 && lane == 0) GM_STAMP(2, i, 3);
            if (++ab == kAcc) ab = 0, aphase ^= 1;
        }
        if (lane == 0) bulk_wait_all();
    } else if (QF && QT) {
        // Converters over the TMA-staged V: thread ct owns items i = ct + j * (32 * kConvWarps)
        // of the stage's kRowsPerTile x (BK / 16) chunk grid; 32 B of V in, 16 B of A out.
        constexpr int kCh = BK / 16, kItems = kRowsPerTile * kCh / (32 * kConvWarps);
        const int ct = threadIdx.x - 32 * (2 + kEpiWarps);
        griddep_wait();  // vmax comes from the activation pass
        const QuantParams qp = qparams_warp(*qf.vmax, qf.bits, qf.qtab);
        if (blockIdx.x == 0 && ct == 0) *qf.qp_out = qp;
        const int npairs = ((units - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x)) * nk;
        auto run = [&](auto quant) {
            int stage = 0;
            uint32_t phase = 0;
            for (int s2 = 0; s2 < npairs; ++s2) {
                ptx::mbar_wait_sleep<100>(&vfull[stage], phase);  // (the producer waited for the stage to be free)
                if (ct == 0) GM_STAMP(3, s2, 0);
                const uint8_t* v_st = sV + stage * kVStageBytes;
                uint8_t* a_st = sA + stage * kRowsPerTile * BK;
#pragma unroll
                for (int j = 0; j < kItems; ++j) {
                    const int i = ct + j * (32 * kConvWarps);
                    const int r = i / kCh, qc = i % kCh;
                    const uint4* src = reinterpret_cast<const uint4*>(v_st + r * (BK * 2) + qc * 32);
                    const uint4 a = src[0], b = src[1];
                    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                    uint32_t o[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e)  // two int16x2 words -> four int8 in one word
                        o[e] = pack_q4(w[2 * e], w[2 * e + 1], quant);
                    const int sw = BK == 128 ? (qc ^ (r & 7)) : (qc ^ ((r >> 1) & 3));
                    *reinterpret_cast<uint4*>(a_st + r * BK + (sw << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
                }
                fence_async_smem();  // generic-proxy stores -> visible to the tensor core (async proxy)
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&full[stage]);
                if (ct == 0) GM_STAMP(3, s2, 1);
                if (++stage == STAGES) stage = 0, phase ^= 1;
            }
        };
        if (qp.exact && qp.shift >= 33) {  // one mad.hi + shift per value (common.cuh)
            const int mul = int(qp.mul), c = 1 << (qp.shift - 33), sh = qp.shift - 32;
            run([=](int v) { return quant_hi32(v, mul, c, sh); });
        } else if (qp.exact) {
            const int mul = int(qp.mul);
            const long long half = 1ll << (qp.shift - 1);
            const int shift = qp.shift;
            run([=](int v) { return quant_fast(v, mul, half, shift); });
        } else {  // (zero-filled padding quantizes to 0: no saturations from it)
            run([&](int v) { return clamp_q(exact_q(v, qp.sa), qp.qmax, qf.sat); });
        }
    } else if (QF) {
        // Converters: thread ct owns items i = ct + j * (32 * kConvWarps) of a stage's
        // kRowsPerTile x (BK / 16) chunk grid (row r = i / (BK / 16), chunk q = i % (BK / 16)).
        constexpr int kCh = BK / 16, kItems = kRowsPerTile * kCh / (32 * kConvWarps);
        const int ct = threadIdx.x - 32 * (2 + kEpiWarps);
        griddep_wait();  // V and vmax come from the activation pass
        const QuantParams qp = qparams_warp(*qf.vmax, qf.bits, qf.qtab);
        if (blockIdx.x == 0 && ct == 0) *qf.qp_out = qp;
        // (u, kc) pairs in issue order; the loads of pair s + 1 are in flight while pair s
        // is converted (register double buffer).
        const int npairs = ((units - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x)) * nk;
        auto load = [&](int s, uint4 (&va)[kItems], uint4 (&vb)[kItems]) {
            const int u = int(blockIdx.x) + (s / nk) * int(gridDim.x), kc = s % nk;
            int ob, tb, f;
            unit_of(u, n_ob, n_tb, F, g.p24 == 2, ob, tb, f);
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                const int i = ct + j * (32 * kConvWarps);
                const int r = i / kCh, qc = i % kCh;
                const int t = tb * kRowsPerTile + r, c = kc * BK + qc * 16;
                va[j] = vb[j] = make_uint4(0, 0, 0, 0);
                if (s < npairs && t < g.T && c < g.C) {
                    const uint4* src = reinterpret_cast<const uint4*>(qf.v + (size_t(f) * g.Tpad + t) * g.Cpad + c);
                    va[j] = __ldg(src);
                    vb[j] = __ldg(src + 1);
                }
            }
        };
        auto run = [&](auto quant) {
            uint4 ca[kItems], cb[kItems], na[kItems], nb[kItems];
            load(0, ca, cb);
            int stage = 0;
            uint32_t phase = 0;
            for (int s = 0; s < npairs; ++s) {
                load(s + 1, na, nb);
                const int kc = s % nk;
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* a_st = sA + stage * kRowsPerTile * BK;
#pragma unroll
                for (int j = 0; j < kItems; ++j) {
                    const int i = ct + j * (32 * kConvWarps);
                    const int r = i / kCh, qc = i % kCh;
                    const int valid = g.C - (kc * BK + qc * 16);  // channels >= C (and rows >= T, loaded as 0) give 0
                    uint32_t w[8] = {ca[j].x, ca[j].y, ca[j].z, ca[j].w, cb[j].x, cb[j].y, cb[j].z, cb[j].w};
                    if (valid < 16) {  // the channel tail of the last chunk: V there is not defined
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (e >= valid) w[e >> 1] &= ~(0xffffu << (16 * (e & 1)));
                    }
                    uint32_t o[4];  // (quant(0) == 0: no saturation from padding)
#pragma unroll
                    for (int e = 0; e < 4; ++e) o[e] = pack_q4(w[2 * e], w[2 * e + 1], quant);
                    const int sw = BK == 128 ? (qc ^ (r & 7)) : (qc ^ ((r >> 1) & 3));
                    *reinterpret_cast<uint4*>(a_st + r * BK + (sw << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
                }
                fence_async_smem();  // generic-proxy stores -> visible to the tensor core (async proxy)
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&full[stage]);
                if (++stage == STAGES) stage = 0, phase ^= 1;
#pragma unroll
                for (int j = 0; j < kItems; ++j) ca[j] = na[j], cb[j] = nb[j];
            }
        };
        if (qp.exact && qp.shift >= 33) {  // CTA-uniform: one specialised loop per quantizer path
            const int mul = int(qp.mul), c = 1 << (qp.shift - 33), sh = qp.shift - 32;
            run([=](int v) { return quant_hi32(v, mul, c, sh); });
        } else if (qp.exact) {
            const int mul = int(qp.mul);
            const long long half = 1ll << (qp.shift - 1);
            const int shift = qp.shift;
            run([=](int v) { return quant_fast(v, mul, half, shift); });
        } else {
            run([&](int v) { return clamp_q(exact_q(v, qp.sa), qp.qmax, qf.sat); });
        }
    }
    __syncthreads();
#ifdef GM_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0 && units > 40 * int(gridDim.x)) {
        const long long t0 = s_trace[(0 * 32 + 8) * 4 + 0];
        for (int u2 = 8; u2 < 28; ++u2)
            printf("g%2d prod: free %6lld issued %6lld | conv: vfull %6lld done %6lld | mma: tempty %6lld full %6lld committed %6lld | epi: tfull %6lld ld %6lld bufready %6lld released %6lld\n",
                   u2, s_trace[(0 * 32 + u2) * 4 + 0] - t0, s_trace[(0 * 32 + u2) * 4 + 1] - t0,
                   s_trace[(3 * 32 + u2) * 4 + 0] - t0, s_trace[(3 * 32 + u2) * 4 + 1] - t0,
                   s_trace[(1 * 32 + u2) * 4 + 0] - t0, s_trace[(1 * 32 + u2) * 4 + 1] - t0, s_trace[(1 * 32 + u2) * 4 + 2] - t0,
                   s_trace[(2 * 32 + u2) * 4 + 0] - t0, s_trace[(2 * 32 + u2) * 4 + 1] - t0, s_trace[(2 * 32 + u2) * 4 + 2] - t0,
                   s_trace[(2 * 32 + u2) * 4 + 3] - t0);
    }
#endif
    tl_mark(kTlGemm, 2);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, kTmemCols);
    }
}

// ============================================================================ host
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

bool make_tmap_3d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base, uint64_t d0, uint64_t d1,
                  uint64_t d2, uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw, uint64_t plane_rows = 0) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0 * esize, d0 * (plane_rows ? plane_rows : d1) * esize};
    cuuint32_t box[3] = {b0, b1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The GEMM's P maps: int32 [F][Tpad][OCpad] boxes of 32 x 32 (rows x oc), 128B-swizzled; or
// 24-bit P as rows of 3*OCpad bytes (byte planes b0 | b1 | b2 of OCpad bytes each): one byte
// map, box 32 B x 32 rows, 32B swizzle, stored once per plane.
bool make_p_maps(CUtensorMap* m, CUtensorMap* m2, CUtensorMap* m3, int32_t* P, const ConvGeom& g, int F, int rows) {
    *m2 = CUtensorMap{};
    *m3 = CUtensorMap{};
    if (g.p24 == 2) {  // unit-major: box [planes 0-1][8 tile groups][128 B] per f (and plane 2 alone), 128B-swizzled staging
        return make_pu_map(m2, P, g, F, 8, 1, true, 2) && make_pu_map(m3, P, g, F, 8, 1, true) &&
               make_tmap_3d(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, P, uint64_t(g.OCpad) * 3, rows, F, 32, 32,
                            CU_TENSOR_MAP_SWIZZLE_32B);
    }
    if (!g.p24)
        return make_tmap_3d(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, P, g.OCpad, rows, F, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    return make_tmap_3d(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, P, uint64_t(g.OCpad) * 3, rows, F, 32, 32,
                        CU_TENSOR_MAP_SWIZZLE_32B);
}

int sm_count() { return device_sm_count(); }
}  // namespace

bool make_pu_map(CUtensorMap* m, void* P, const ConvGeom& g, int F, int box_tg, int box_f, bool swizzle128,
                 int box_planes) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t ntg = cuuint64_t(g.Tpad) / kUnitTiles;
    cuuint64_t dims[5] = {128, ntg, cuuint64_t(F), 3, cuuint64_t(g.OCpad) / kUnitOc};
    cuuint64_t strides[4] = {128, ntg * 128, cuuint64_t(F) * ntg * 128, 3 * cuuint64_t(F) * ntg * 128};
    cuuint32_t box[5] = {128, cuuint32_t(box_tg), cuuint32_t(box_f), cuuint32_t(box_planes), 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, P, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

template <int BN, int BK, int STAGES, bool QF, bool QT = false>
cudaError_t gemm_launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& p, const CUtensorMap& p2,
                        const CUtensorMap& p3, const ConvGeom& g, int F, const QFuse& qf, cudaStream_t st, bool pdl,
                        void* p_raw) {
    const size_t smem = size_t(STAGES) * (kRowsPerTile + BN) * BK + (QT ? size_t(STAGES) * kRowsPerTile * BK * 2 : 0) +
                        size_t(kEpiWarps) * kEpiBufs * kEpiBoxBytes + 1024 + 256
#ifdef GM_TRACE
                        + 4200
#endif
        ;
    auto kern = k_gemm<BN, BK, STAGES, QF, QT>;
    static SmemOptIn opt_in;
    if (cudaError_t e = opt_in.ensure(kern, smem); e != cudaSuccess) return e;
    const int n_tb = g.Tpad / kRowsPerTile, n_ob = g.OCpad / BN;
    const int units = F * n_tb * n_ob;
    // CTAs per SM bounded by shared memory and by TMEM (2*BN columns each of 512).
    constexpr int kAcc = gemm_acc<BN, BK, STAGES, QT>();
    constexpr int kTmemCols = kAcc * BN <= 128 ? 128 : (kAcc * BN <= 256 ? 256 : 512);
    int per_sm = int((227 * 1024) / smem);
    per_sm = per_sm < 1 ? 1 : per_sm;
    per_sm = per_sm > 512 / kTmemCols ? 512 / kTmemCols : per_sm;
    per_sm = per_sm > 2 ? 2 : per_sm;
    int resident = sm_count() * per_sm;
    if (const char* e = std::getenv("SFC_GEMM_GRID")) {  // experiment knob: cap the persistent grid
        const int cap = std::atoi(e);
        if (cap > 0 && cap < resident) resident = cap;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(units < resident ? units : resident);
    cfg.blockDim = dim3(gemm_threads<QF>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    ConvGeom gk = g;
    if (g.p24 == 2) {  // unit-major P: tile-block-major unit order unless SFC_GEMM_FMAJOR=1 (A/B knob)
        const char* e = std::getenv("SFC_GEMM_FMAJOR");
        if (!(e && e[0] == '1')) gk.p24 = 3;  // (3: unit-major P, tile-block-major order)
    }
    return cudaLaunchKernelEx(&cfg, kern, a, b, p, p2, p3, n_tb, n_ob, F, g.Cpad / BK, gk, qf, static_cast<uint8_t*>(p_raw));
}

template <int BK, int STAGES, bool QF>
cudaError_t gemm_by_bn(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& p, const CUtensorMap& p2,
                       const CUtensorMap& p3, const ConvGeom& g, int F, const QFuse& qf, cudaStream_t st, bool pdl,
                       void* p_raw) {
    if (g.BN == 64) return gemm_launch<64, BK, STAGES, QF>(a, b, p, p2, p3, g, F, qf, st, pdl, p_raw);
    if (g.BN == 128) return gemm_launch<128, BK, STAGES, QF>(a, b, p, p2, p3, g, F, qf, st, pdl, p_raw);
    return gemm_launch<256, BK, STAGES, QF>(a, b, p, p2, p3, g, F, qf, st, pdl, p_raw);
}

template <bool QF>
cudaError_t gemm_dispatch(const int8_t* vqA, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, const QFuse& qf,
                          cudaStream_t st, bool pdl) {
    CUtensorMap ta, tb, tp, tp2, tp3;
    const CUtensorMapSwizzle sw = g.BK == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    // (QF: the A map is unused; it is built over the filters only to keep one kernel signature)
    if (!make_tmap_3d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, QF ? static_cast<const void*>(uqB) : vqA, g.Cpad,
                      QF ? g.OCpad : g.Tpad, F, g.BK, QF ? g.BN : kRowsPerTile, sw) ||
        !make_tmap_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, uqB, g.Cpad, g.OCpad, F, g.BK, g.BN, sw) ||
        !make_p_maps(&tp, &tp2, &tp3, P, g, F, g.Tpad))
        return cudaErrorInvalidValue;
    const int nk = g.Cpad / g.BK;
    if (g.BK == 128)
        return nk <= 2 ? gemm_by_bn<128, 2, QF>(ta, tb, tp, tp2, tp3, g, F, qf, st, pdl, P)
                       : gemm_by_bn<128, 3, QF>(ta, tb, tp, tp2, tp3, g, F, qf, st, pdl, P);
    return nk <= 2 ? gemm_by_bn<64, 2, QF>(ta, tb, tp, tp2, tp3, g, F, qf, st, pdl, P)
                   : gemm_by_bn<64, 4, QF>(ta, tb, tp, tp2, tp3, g, F, qf, st, pdl, P);
}
}  // namespace

cudaError_t launch_gemm(const int8_t* vqA, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, cudaStream_t st,
                        bool pdl) {
    return gemm_dispatch<false>(vqA, uqB, P, g, F, QFuse{}, st, pdl);
}

cudaError_t launch_gemm_rows(const int8_t* vqA, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, int t0,
                             int tcpad, cudaStream_t st, bool pdl) {
    // A: rows [t0, t0 + tcpad) of every frequency plane of vq (rows past the planes' Tpad
    // read as zeros); P: a buffer of tcpad rows per frequency
    CUtensorMap ta, tb, tp, tp2{}, tp3{};
    const CUtensorMapSwizzle sw = g.BK == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    const int arows = tcpad < g.Tpad - t0 ? tcpad : g.Tpad - t0;
    if (!make_tmap_3d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, vqA + size_t(t0) * g.Cpad, g.Cpad, arows, F, g.BK,
                      kRowsPerTile, sw, g.Tpad) ||
        !make_tmap_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, uqB, g.Cpad, g.OCpad, F, g.BK, g.BN, sw) ||
        !make_tmap_3d(&tp, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, P, g.OCpad, tcpad, F, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
    ConvGeom gc = g;
    gc.Tpad = tcpad;
    const int nk = g.Cpad / g.BK;
    const QFuse none{};
    if (g.BK == 128)
        return nk <= 2 ? gemm_by_bn<128, 2, false>(ta, tb, tp, tp2, tp3, gc, F, none, st, pdl, P)
                       : gemm_by_bn<128, 3, false>(ta, tb, tp, tp2, tp3, gc, F, none, st, pdl, P);
    return nk <= 2 ? gemm_by_bn<64, 2, false>(ta, tb, tp, tp2, tp3, gc, F, none, st, pdl, P)
                   : gemm_by_bn<64, 4, false>(ta, tb, tp, tp2, tp3, gc, F, none, st, pdl, P);
}

cudaError_t launch_gemm_qfused(const QFuse& q, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, cudaStream_t st,
                               bool pdl) {
    return gemm_dispatch<true>(nullptr, uqB, P, g, F, q, st, pdl);
}

cudaError_t launch_gemm_qtma(const QFuse& q, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, cudaStream_t st,
                             bool pdl) {
    // V [F][Tpad][Cpad] int16 seen as (C, T, F): channels >= C and rows >= T read as zero
    auto fn = encode_fn();
    if (!fn) return cudaErrorInvalidValue;
    CUtensorMap tv, tb, tp, tp2, tp3;
    cuuint64_t dims[3] = {cuuint64_t(g.C), cuuint64_t(g.T), cuuint64_t(F)};
    cuuint64_t strides[2] = {cuuint64_t(g.Cpad) * 2, cuuint64_t(g.Cpad) * g.Tpad * 2};
    cuuint32_t box[3] = {cuuint32_t(g.BK), cuuint32_t(kRowsPerTile), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (fn(&tv, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<int16_t*>(q.v), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    const CUtensorMapSwizzle sw = g.BK == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    if (!make_tmap_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, uqB, g.Cpad, g.OCpad, F, g.BK, g.BN, sw) ||
        !make_p_maps(&tp, &tp2, &tp3, P, g, F, g.Tpad))
        return cudaErrorInvalidValue;
    // stages: A + B + V per stage plus the 64 KB of epilogue boxes within 227 KB -- two at
    // BK = 128, four at BK = 64 with BN <= 128 (the single-K-chunk
    // 64-channel layers: more units' V tiles in flight to hide the load latency)
    if (g.BK == 128) {
        if (g.BN == 64) return gemm_launch<64, 128, 2, true, true>(tv, tb, tp, tp2, tp3, g, F, q, st, pdl, P);
        if (g.BN == 128) return gemm_launch<128, 128, 2, true, true>(tv, tb, tp, tp2, tp3, g, F, q, st, pdl, P);
        return gemm_launch<256, 128, 2, true, true>(tv, tb, tp, tp2, tp3, g, F, q, st, pdl, P);
    }
    if (g.BN == 64) return gemm_launch<64, 64, 4, true, true>(tv, tb, tp, tp2, tp3, g, F, q, st, pdl, P);
    if (g.BN == 128) return gemm_launch<128, 64, 4, true, true>(tv, tb, tp, tp2, tp3, g, F, q, st, pdl, P);
    return gemm_launch<256, 64, 2, true, true>(tv, tb, tp, tp2, tp3, g, F, q, st, pdl, P);
}

SFC_TL_UNIT_READER(tl_read_gemm)

}  // namespace sfcb200
