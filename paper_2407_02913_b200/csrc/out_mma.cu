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
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "devcache.hpp"
#include "ptx.cuh"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"

namespace sfcb200 {

namespace {
constexpr int kOmParts = 3;                      // output parts (TMEM column groups of W rows)
constexpr int kOmAWarps = 8;                     // TMEM -> staging warps, two per lane quarter
constexpr int kOmBWarps = 12;                    // staging -> global store warps
constexpr int kOmProdWarps = 2;                  // producers, alternating units (~1800 cycles of issue per unit)
constexpr int kOmMmaWarps = 2;                   // MMA issuers, alternating units (~1000 cycles of issue per unit)
constexpr int kOmFirstA = kOmProdWarps + kOmMmaWarps, kOmFirstB = kOmFirstA + kOmAWarps;
constexpr int kOmThreads = 32 * (kOmFirstB + kOmBWarps);
constexpr int kOmMaxOc = 1024;  // per-channel scales kept in shared memory
constexpr int kOmSparseRows = 8;  // sparse plane 2: flagged rows per unit loaded one by one (more: the box + fix-up)

template <int V>
struct Om {
    static constexpr int F = Tab<V>::F, K = Tab<V>::K, M = Tab<V>::M, MM = M * M;
    static constexpr int KP = (F + 31) / 32 * 32;      // frequencies padded to the MMA K step
    static constexpr int KB = (KP + 127) / 128;        // 128-byte K blocks of W
    static constexpr int PART = (MM + kOmParts - 1) / kOmParts;  // outputs per epilogue part (last: the rest)
    static constexpr int NP = (PART + 7) / 8 * 8;      // W rows (TMEM columns) per part
    static constexpr int N = (kOmParts * NP + 15) / 16 * 16;  // MMA N: 32 / 48 / 80
    // a plane's F rows, padded to the 1 KB swizzle atom; the K steps' rows F .. KP - 1 run into the
    // next plane / stage / W (any bytes: their W columns are zero)
    static constexpr uint32_t PLANE = (uint32_t(F) * 128 + 1023) / 1024 * 1024;
    static constexpr uint32_t STAGE = 3 * PLANE;
    static constexpr int FRING = 4;                    // sparse plane 2: units of flag bytes in flight (cp.async)
    static constexpr int ROW = kUnitTiles * M;         // staged columns per (oc, t1): 4 tiles x M
    static constexpr int OCS = M * ROW + 2;            // staged words per output channel, at most (see k_out_mma)
    // accumulator buffers (three N-column accumulators each): the MMA -> commit -> epilogue ->
    // release loop spans NACC units, and its latency, not its work, bounds the kernel
#ifdef OM_NACC
    static constexpr int NACC = OM_NACC;
#else
    static constexpr int NACC = 512 / (3 * N) >= 4 ? 4 : 512 / (3 * N);
#endif
    static constexpr int TMEM_COLS = 512;
    static_assert(NACC >= 2 && NACC * 3 * N <= 512, "the accumulator buffers must fit TMEM");
    static constexpr size_t W_BYTES = size_t(KB) * N * 128;
    static constexpr size_t Y_BYTES = size_t(kUnitOc) * OCS * 4;  // one staging buffer (two are used)
    static constexpr size_t FLAG_BYTES = size_t(kOmProdWarps) * FRING * KP * 8;  // [producer][FRING][KP] flag words (8 tile groups each)
    static constexpr size_t FIXED = 1024 + W_BYTES + 2 * Y_BYTES + kOmMaxOc * 12 + 512 + FLAG_BYTES + 4 * KP
#ifdef OM_TRACE
                                    + 4200
#endif
        ;
#ifdef OM_STAGES  // experiment builds (make EXTRA=-DOM_STAGES=n)
    static constexpr int STAGES = OM_STAGES;
#else
    // bulk-copy pipeline depth: the stage ring's round trip (free -> issue -> HBM latency -> MMAs)
    // bounds the kernel, so as many stages as fit
    static constexpr int STAGES = (227 * 1024 - FIXED) / STAGE >= 4 ? 4 : int((227 * 1024 - FIXED) / STAGE);
#endif
    static_assert(STAGES >= 2, "at least two stages must fit");
    static constexpr size_t SMEM = FIXED + STAGES * size_t(STAGE);
};

#ifdef OM_TRACE  // experiment build: clock stamps of CTA 0's first units per role, printed at exit
#define OM_STAMP(role, unit, k) do { if (blockIdx.x == 0 && (unit) < 32) s_trace[((role) * 32 + (unit)) * 4 + (k)] = clock64(); } while (0)
#else
#define OM_STAMP(role, unit, k) do { } while (0)
#endif

struct TileInfo {
    long long base;  // output offset of the tile's (oc 0, t1 0, t2 0) element (channel oc0 of the unit)
    int rows, cols;  // valid output rows / columns (0 rows: padding tile)
};

// Unit u = tg * n_ob + ob walked with stride gridDim.x without a division per unit.
struct UnitWalk {
    int ob, tg, sob, stg, n_ob;
    __device__ __forceinline__ UnitWalk(int u0, int stride, int n_ob_) : n_ob(n_ob_) {
        ob = u0 % n_ob, tg = u0 / n_ob, sob = stride % n_ob, stg = stride / n_ob;
    }
    __device__ __forceinline__ void next() {
        ob += sob, tg += stg;
        if (ob >= n_ob) ob -= n_ob, ++tg;
    }
};

__device__ __forceinline__ void named_bar_epi() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kOmBWarps) : "memory"); }

// MK: compile-time output set (bits: 1 y32, 2 y64, 4 f32, 8 f64, 16 i8); 0 = read o at run time
template <int V, int MK>
__global__ void __launch_bounds__(kOmThreads, 1)
    k_out_mma(const __grid_constant__ CUtensorMap tmP, ConvGeom g, const QuantParams* __restrict__ qpp,
              const double* __restrict__ sf, OutPtrs o, int n_ob, int n_tg, int units,
              const uint8_t* __restrict__ p_raw) {
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
    uint64_t* s_fring = reinterpret_cast<uint64_t*>(s_scalef + kOmMaxOc);  // [FRING][KP] flag words in flight
    uint8_t* s_flag = reinterpret_cast<uint8_t*>(s_fring + kOmProdWarps * C::FRING * C::KP);  // [STAGES][KP] flag bytes (fix-up mode)
    uint64_t* full = reinterpret_cast<uint64_t*>(s_flag + 4 * C::KP);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + C::NACC;
    uint64_t* yfull = tempty + C::NACC;   // staging buffer filled by the A warps
    uint64_t* yempty = yfull + 2;         // ... read by the B warps
    TileInfo* s_tile = reinterpret_cast<TileInfo*>(yempty + 2);  // 2 x [kUnitTiles]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_tile + 2 * kUnitTiles);
    uint32_t* s_kmask = tmem_holder + 1;  // [STAGES]: K steps of plane 2 holding flagged rows (sparse plane 2)
#ifdef OM_TRACE
    long long* s_trace = reinterpret_cast<long long*>((reinterpret_cast<uintptr_t>(s_kmask + 4) + 15) & ~uintptr_t(15));
    int tu = 0;
#endif
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // staged words per output channel: odd (conflict-free staging) for single columns, even
    // for the 8-byte pair loads
    constexpr int OCSK = (C::M % 2 == 0 && MK == 16) ? C::M * C::ROW + 2 : C::M * C::ROW + 1;
    // experiment knob SFC_OM_DEBUG (bits): 1 skips the TMEM phase, 2 the store phase, 4 the MMAs, 8 the loads
    const int dbg = o.pairs >> 8;
    tl_mark(kTlOutput, 0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) ptx::mbar_init(&full[s], 1), ptx::mbar_init(&empty[s], 1);
        for (int i = 0; i < C::NACC; ++i) ptx::mbar_init(&tfull[i], 1), ptx::mbar_init(&tempty[i], kOmAWarps);
        for (int i = 0; i < 2; ++i) ptx::mbar_init(&yfull[i], kOmAWarps), ptx::mbar_init(&yempty[i], kOmBWarps);
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
    // sparse plane 2: the rows of plane 2 start as zeros; the producer then zeroes only rows it
    // loaded earlier and that are no longer flagged (dirty rows)
    for (int i = threadIdx.x; i < C::STAGES * C::F * 8; i += kOmThreads) {
        const int st_ = i / (C::F * 8), r_ = i % (C::F * 8);
        reinterpret_cast<uint4*>(sA + size_t(st_) * C::STAGE + 2 * C::PLANE)[r_] = make_uint4(0, 0, 0, 0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // W, zeros (generic stores) -> tensor core
    if (warp == kOmProdWarps) ptx::tmem_alloc(tmem_holder, C::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    griddep_wait();  // P and the activation scale are complete
    tl_mark(kTlOutput, 1);
    griddep_launch_dependents();

    if (warp < kOmProdWarps) {
        // Producers (NPROD of them, unit n = pm (mod NPROD) each; a stage always belongs to one).
        // Producer.  Dense P: lane 0 issues one TMA box per plane.  Sparse plane 2 (g.p2s): every
        // lane owns the rows f = lane + 32 j of plane 2 -- a 128-byte bulk copy when the GEMM
        // flagged the row, zeros otherwise (only in K steps that hold a flagged row, and in K
        // step 0, which always runs); the next unit's flags are in flight during the wait.
        constexpr int KS = C::KP / 32;
        constexpr int NPROD = C::STAGES % kOmProdWarps == 0 ? kOmProdWarps : 1;
        const int pm = warp;
#ifdef OM_TRACE
        tu = pm;
#endif
        const int u0 = pm < NPROD ? int(blockIdx.x) + pm * int(gridDim.x) : units, ustep = NPROD * int(gridDim.x);
        if (lane == 0) ptx::tma_prefetch(&tmP);
        // the flag words (8 tile groups per (oc block, tile group / 8, f)) of the next FRING units
        // are always in flight: cp.async into a ring, one group per unit, so the producer never
        // waits an HBM round trip between a stage becoming free and its loads being issued
        const uint8_t* flags = p_raw + p2_flags_offset(C::F, g.Tpad, g.OCpad);
        auto fetch_flags = [&](int u, int ob, int tg, int slot) {
            if (u < units) {
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    const int f = lane + 32 * j;
                    if (f < C::F)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                                         ptx::smem_u32(s_fring + (pm * C::FRING + slot) * C::KP + f)),
                                     "l"(flags + p2_flag_index(ob, tg & ~7, f, g.Tpad, C::F))
                                     : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        UnitWalk uw(u0, ustep, n_ob);   // this iteration's unit
        UnitWalk uf(u0, ustep, n_ob);   // the unit whose flags are fetched
        int fslot = 0;
        if (g.p2s) {
#pragma unroll
            for (int d = 0; d < C::FRING - 1; ++d) {
                fetch_flags(u0 + d * ustep, uf.ob, uf.tg, d);
                uf.next();
            }
        }
        uint32_t fl[KS] = {};
        uint32_t dirty[C::STAGES] = {};  // bit j: this lane's row lane + 32 j of the stage's plane 2 holds data
        int stage = pm;
        uint32_t phase = 0;
        for (int u = u0; u < units; u += ustep) {
            const int ob = uw.ob, tg = uw.tg;
            uw.next();
            if (g.p2s) {
                fetch_flags(u + (C::FRING - 1) * ustep, uf.ob, uf.tg, (fslot + C::FRING - 1) % C::FRING);
                uf.next();
                asm volatile("cp.async.wait_group %0;" ::"n"(C::FRING - 1) : "memory");
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    const int f = lane + 32 * j;
                    fl[j] = f < C::F ? reinterpret_cast<const uint8_t*>(s_fring + (pm * C::FRING + fslot) * C::KP + f)[tg & 7] : 0u;
                }
                fslot = (fslot + 1) % C::FRING;
            }
            ptx::mbar_wait(&empty[stage], phase ^ 1);
#ifdef OM_TRACE
            if (lane == 0) OM_STAMP(0, tu, 0);
#endif
            uint8_t* dst = sA + size_t(stage) * C::STAGE;
            uint32_t kmask = 0;
            int cnt = 0;
            if (g.p2s) {
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    const uint32_t b = __ballot_sync(0xffffffffu, fl[j] != 0);
                    kmask |= b ? 1u << j : 0u;
                    cnt += __popc(b);
                }
            }
            if (dbg & 8) {
                if (lane == 0) {
                    s_kmask[stage] = 0x7fffffffu;
                    ptx::mbar_arrive(&full[stage]);
                }
            } else if (!g.p2s || cnt == C::F) {
#pragma unroll
                for (int s2 = 0; s2 < C::STAGES; ++s2)
                    if (s2 == stage) dirty[s2] = 0xffffffffu;
                if (lane == 0) {
                    s_kmask[stage] = 0x7fffffffu;
                    ptx::mbar_expect_tx(&full[stage], 3u * C::F * 128);
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl) ptx::tma_load_5d(dst + pl * C::PLANE, &tmP, &full[stage], 0, tg, 0, pl, ob);
                }
            } else if (cnt > kOmSparseRows) {
                // many flagged rows: the whole plane-2 box (unwritten rows hold stale bytes); the MMA
                // warp zeroes the unflagged rows once it has landed (bit 31 of the mask)
#pragma unroll
                for (int s2 = 0; s2 < C::STAGES; ++s2)
                    if (s2 == stage) dirty[s2] = 0xffffffffu;
#pragma unroll
                for (int j = 0; j < KS; ++j) s_flag[stage * C::KP + lane + 32 * j] = uint8_t(fl[j]);
                __syncwarp();
                if (lane == 0) {
                    s_kmask[stage] = 0xffffffffu;
                    ptx::mbar_expect_tx(&full[stage], 3u * C::F * 128);
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl) ptx::tma_load_5d(dst + pl * C::PLANE, &tmP, &full[stage], 0, tg, 0, pl, ob);
                }
            } else {
                kmask |= 1u;
                uint32_t dm = 0;
#pragma unroll
                for (int s2 = 0; s2 < C::STAGES; ++s2)
                    if (s2 == stage) dm = dirty[s2];
                bool zeroed = false;
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    const int f = lane + 32 * j;
                    if (!((kmask >> j) & 1u) || f >= C::F) continue;
                    uint8_t* row = dst + 2 * C::PLANE + f * 128;
                    if (fl[j]) {
                        ptx::bulk_load(row, p_raw + pu_offset(ob, tg, 2, f, n_tg, C::F), 128, &full[stage]);
                        dm |= 1u << j;
                    } else if ((dm >> j) & 1u) {  // loaded by an earlier unit, not flagged now
#pragma unroll
                        for (int c = 0; c < 8; ++c) reinterpret_cast<uint4*>(row)[c] = make_uint4(0, 0, 0, 0);
                        dm &= ~(1u << j);
                        zeroed = true;
                    }
                }
#pragma unroll
                for (int s2 = 0; s2 < C::STAGES; ++s2)
                    if (s2 == stage) dirty[s2] = dm;
                if (__any_sync(0xffffffffu, zeroed))
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the zero rows -> tensor core
                __syncwarp();
                if (lane == 0) {
                    s_kmask[stage] = kmask;
                    ptx::mbar_expect_tx(&full[stage], (2u * C::F + uint32_t(cnt)) * 128);
#pragma unroll
                    for (int pl = 0; pl < 2; ++pl) ptx::tma_load_5d(dst + pl * C::PLANE, &tmP, &full[stage], 0, tg, 0, pl, ob);
                }
            }
#ifdef OM_TRACE
            if (lane == 0) OM_STAMP(0, tu, 1);
            tu += NPROD;
#endif
            stage += NPROD;
            if (stage >= C::STAGES) stage -= C::STAGES, phase ^= 1;
        }
    } else if (warp < kOmFirstA) {
        // MMA issuers: warp kOmProdWarps + m takes the units n = m (mod kOmMmaWarps) of this CTA
        constexpr uint32_t id_u = ptx::idesc_i8_amn(128, C::N, false), id_s = ptx::idesc_i8_amn(128, C::N, true);
        // descriptors once: the address field is the low 14 bits (address >> 4), so a plane / K step /
        // stage offset is one 32-bit add
        const uint64_t ad0 = ptx::smem_desc_mn128(ptx::smem_u32(sA));
        uint64_t wd[C::KP / 32];
#pragma unroll
        for (int ks = 0; ks < C::KP / 32; ++ks)
            wd[ks] = ptx::smem_desc_kmajor(ptx::smem_u32(sW) + (ks / 4) * (C::N * 128) + (ks % 4) * 32, 128);
        const int m = warp - kOmProdWarps;
#ifdef OM_TRACE
        tu = m;
#endif
        int stage = m % C::STAGES, ab = m % C::NACC;
        uint32_t phase = 0, aphase = 0;
        for (int u = blockIdx.x + m * gridDim.x; u < units; u += kOmMmaWarps * gridDim.x) {
            ptx::mbar_wait(&tempty[ab], aphase ^ 1);
#ifdef OM_TRACE
            if (lane == 0) OM_STAMP(1, tu, 0);
#endif
            ptx::mbar_wait(&full[stage], phase);
#ifdef OM_TRACE
            if (lane == 0) OM_STAMP(1, tu, 1);
#endif
            const uint32_t km = s_kmask[stage];  // plane-2 K steps to run (bit 0 always set)
            if (km >> 31) {  // fix-up: zero the plane-2 rows the GEMM did not write
                uint8_t* p2 = sA + size_t(stage) * C::STAGE + 2 * C::PLANE;
#pragma unroll
                for (int j = 0; j < C::KP / 32; ++j) {
                    const int f = lane + 32 * j;
                    if (f < C::F && !s_flag[stage * C::KP + f]) {
#pragma unroll
                        for (int c = 0; c < 8; ++c) reinterpret_cast<uint4*>(p2 + f * 128)[c] = make_uint4(0, 0, 0, 0);
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
            }
            if (lane == 0) {
                ptx::tc_fence_after();
                const uint64_t ad = ad0 + uint64_t(uint32_t(stage) * (C::STAGE >> 4));
                const uint32_t dcol = tmem + uint32_t(ab * 3 * C::N);
#pragma unroll
                for (int ks = 0; ks < C::KP / 32; ++ks) {
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl)
                        if ((pl < 2 || ((km >> ks) & 1u)) && !(dbg & 4))
                            ptx::mma_i8(dcol + uint32_t(pl * C::N), ad + uint64_t((pl * C::PLANE + ks * 32 * 128) >> 4),
                                        wd[ks], pl == 2 ? id_s : id_u, ks > 0);
                }
                ptx::mma_commit(&empty[stage]);
                ptx::mma_commit(&tfull[ab]);
            }
            __syncwarp();
#ifdef OM_TRACE
            if (lane == 0) OM_STAMP(1, tu, 2);
            tu += kOmMmaWarps;
#endif
            stage += kOmMmaWarps;
            if (stage >= C::STAGES) stage -= C::STAGES, phase ^= 1;
            ab += kOmMmaWarps;
            if (ab >= C::NACC) ab -= C::NACC, aphase ^= 1;
        }
    } else if (warp < kOmFirstB) {
        // A warps: warp (q, h) reads TMEM lane quarter q = warp & 3 (tile q of the unit, lane = oc), half
        // h of the M * M outputs, recombines the planes and parks y in the staging buffer.
        const int q = warp & 3, h = (warp - kOmFirstA) >> 2;
        const int WO = g.WO, HO = g.HO, plane = HO * WO;
        const int tiles_img = g.th * g.tw;
        const uint32_t bias_on = g.p2s ? 0xffffffffu : 0u;
        UnitWalk uw(blockIdx.x, gridDim.x, n_ob);
        int ab = 0, n = 0;  // accumulator buffer (of NACC), unit counter
        uint32_t aphase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++n) {
            const int ob = uw.ob, tg = uw.tg, yb = n & 1;
            uw.next();
            int* sy = s_y + yb * (C::Y_BYTES / 4);
            ptx::mbar_wait_sleep<100>(&tfull[ab], aphase);
#ifdef OM_TRACE
            if (warp == kOmFirstA && lane == 0) OM_STAMP(2, tu, 0);
#endif
            ptx::mbar_wait_sleep<100>(&yempty[yb], ((n >> 1) & 1) ^ 1);  // the B warps are done with unit n - 2
#ifdef OM_TRACE
            if (warp == kOmFirstA && lane == 0) OM_STAMP(2, tu, 1);
#endif
            ptx::tc_fence_after();
            if (lane == 0 && h == 0) {  // the tile's output window
                const int t = tg * kUnitTiles + q;
                TileInfo ti{0, 0, 0};
                if (t < g.T) {
                    const int b = t / tiles_img, r = t - b * tiles_img, tr = r / g.tw, tc = r - tr * g.tw;
                    ti.base = ((long long)(b) * g.OC + ob * kUnitOc) * plane + (long long)(tr * C::M) * WO + tc * C::M;
                    ti.rows = min(C::M, HO - tr * C::M);
                    ti.cols = min(C::M, WO - tc * C::M);
                }
                s_tile[yb * kUnitTiles + q] = ti;
            }
            int* yr = sy + lane * OCSK + q * C::M;
            if (!(dbg & 1)) {
                // 8-column slots of the parts' TMEM columns; the quarter's two warps take half each
                constexpr int SPP = C::NP / 8, SLOTS = kOmParts * SPP, SPLIT = (SLOTS + 1) / 2;
#pragma unroll
                for (int sl = 0; sl < SLOTS; ++sl) {
                    const int pp = sl / SPP, c0 = (sl % SPP) * 8;                                       // compile time
                    const int cntp = C::MM - pp * C::PART < C::PART ? C::MM - pp * C::PART : C::PART;  // compile time
                    if (c0 >= cntp || (sl < SPLIT) != (h == 0)) continue;
                    int32_t d0[8], d1[8], d2[8];
                    const uint32_t base = tmem + (uint32_t(q * 32) << 16) + uint32_t(ab * 3 * C::N + pp * C::NP + c0);
                    ptx::tmem_ld8(base, d0);
                    ptx::tmem_ld8(base + C::N, d1);
                    ptx::tmem_ld8(base + 2 * C::N, d2);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (c0 + c < cntp) {
                            // y = D0 + 2^8 D1 + 2^16 D2 (exact mod 2^32: |y| < 2^31); sparse plane 2: the
                            // GEMM stored P + 2^15, so y' = y + 2^15 (sum_k A[k][t1]) (sum_l A[l][t2])
                            const int oo = pp * C::PART + c0 + c, t1 = oo / C::M, t2 = oo % C::M;
                            int s1 = 0, s2 = 0;
#pragma unroll
                            for (int k = 0; k < C::K; ++k) s1 += T::a(k, t1), s2 += T::a(k, t2);
                            const uint32_t y = uint32_t(d0[c]) + (uint32_t(d1[c]) << 8) + (uint32_t(d2[c]) << 16) -
                                               (bias_on & (32768u * uint32_t(s1 * s2)));
                            yr[t1 * C::ROW + t2] = int(y);
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();  // the warp's staging stores and TMEM reads are done
            if (lane == 0) {
                ptx::mbar_arrive(&tempty[ab]);
                ptx::mbar_arrive(&yfull[yb]);
            }
#ifdef OM_TRACE
            if (warp == kOmFirstA && lane == 0) OM_STAMP(2, tu, 2);
            ++tu;
#endif
            if (++ab == C::NACC) ab = 0, aphase ^= 1;
        }
    } else {
        // B warps: all 32 * kOmBWarps threads write the staged unit's output rows (4 tiles x M columns
        // per row when the tiles share an image row) with the requested conversions.
        const int et = threadIdx.x - 32 * kOmFirstB;  // 0 .. 32 * kOmBWarps - 1
        const double sa = qpp->sa, rq = o.requant;
        for (int i = et; i < g.OC; i += 32 * kOmBWarps) {
            const double sc = (sa * sf[i]) / double(T::DEN * T::DEN);
            s_scale[i] = sc;
            s_scalef[i] = float(sc);
        }
        named_bar_epi();  // the scales are in place
        const int WO = g.WO, plane = g.HO * WO;
        // column pairs (8-byte shared loads, 2-byte stores) for int8-only outputs of the even-M
        // variants; single columns otherwise (measured: pairs help the int8 layers of configs
        // 3-4, not the int32 outputs of config 5)
        constexpr int PW = (C::M % 2 == 0 && MK == 16) ? 2 : 1;
        constexpr int CPR = C::ROW / PW;                 // column items per staged row
        constexpr int NG = (32 * kOmBWarps) / CPR;       // channel groups of the store phase
        const int x_col = PW * (et % CPR), x_grp = et / CPR, x_tt = x_col / C::M, x_t2 = x_col % C::M;
        int rofs[C::M];  // row offsets t1 * WO
#pragma unroll
        for (int t1 = 0; t1 < C::M; ++t1) rofs[t1] = t1 * WO;
        UnitWalk uw(blockIdx.x, gridDim.x, n_ob);
        int n = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++n) {
            const int ob = uw.ob, sb = n & 1;
            uw.next();
            int* sy = s_y + sb * (C::Y_BYTES / 4);
            TileInfo* st = s_tile + sb * kUnitTiles;
            ptx::mbar_wait_sleep<100>(&yfull[sb], (n >> 1) & 1);
#ifdef OM_TRACE
            if (et == 0) OM_STAMP(3, tu, 0);
#endif
            // stores: thread et keeps a column pair (x, x + 1) = PW (et % (ROW / PW)) of the unit's
            // staged rows (tile x / M, columns t2 (+1) of that tile; pairs for the even M of the
            // 6x6 / 4x4 variants) and walks output channels oc = et / (ROW / PW), + NG, ..., all
            // M rows each (predicated per row); consecutive threads write consecutive columns
            if (et < NG * CPR && !(dbg & 2)) {
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
                        if (MK != 0 && ti.rows == C::M && (PW == 1 || pair)) {
                            // whole tile (every row, this thread's columns valid and aligned): the
                            // compile-time output set without predicates
                            if constexpr ((MK & 1) != 0) {
                                int32_t* d = o.y32 + e0;
#pragma unroll
                                for (int t1 = 0; t1 < C::M; ++t1) {
                                    if constexpr (PW == 2) *reinterpret_cast<int2*>(d + rofs[t1]) = make_int2(ya[t1], yb[t1]);
                                    else d[rofs[t1]] = ya[t1];
                                }
                            }
                            if constexpr ((MK & 2) != 0) {
                                int64_t* d = o.y64 + e0;
#pragma unroll
                                for (int t1 = 0; t1 < C::M; ++t1) {
                                    d[rofs[t1]] = ya[t1];
                                    if constexpr (PW == 2) d[rofs[t1] + 1] = yb[t1];
                                }
                            }
                            if constexpr ((MK & 4) != 0) {
                                float* d = o.f32 + e0;
#pragma unroll
                                for (int t1 = 0; t1 < C::M; ++t1) {
                                    const float fa = __int2float_rn(ya[t1]) * scf;
                                    if constexpr (PW == 2)
                                        *reinterpret_cast<float2*>(d + rofs[t1]) = make_float2(fa, __int2float_rn(yb[t1]) * scf);
                                    else d[rofs[t1]] = fa;
                                }
                            }
                            if constexpr ((MK & 8) != 0) {
                                double* d = o.f64 + e0;
#pragma unroll
                                for (int t1 = 0; t1 < C::M; ++t1) {
                                    d[rofs[t1]] = double(ya[t1]) * sc;
                                    if constexpr (PW == 2) d[rofs[t1] + 1] = double(yb[t1]) * sc;
                                }
                            }
                            if constexpr ((MK & 16) != 0) {
                                int8_t* d = o.i8 + e0;
                                if (fabs(sc * rq) < 1.0) {  // |y sc rq| < 2^31: conversions on the fp64 add pipe
#pragma unroll
                                    for (int t1 = 0; t1 < C::M; ++t1) {
                                        const int qa = requant_i8_small(ya[t1], sc, rq);
                                        if constexpr (PW == 2) {
                                            const int qb = requant_i8_small(yb[t1], sc, rq);
                                            *reinterpret_cast<uint16_t*>(d + rofs[t1]) = uint16_t(__byte_perm(uint32_t(qa), uint32_t(qb), 0x0040));
                                        } else {
                                            d[rofs[t1]] = int8_t(qa);
                                        }
                                    }
                                } else {
#pragma unroll
                                    for (int t1 = 0; t1 < C::M; ++t1) {
                                        const int qa = requant_i8(double(ya[t1]) * sc * rq);
                                        if constexpr (PW == 2) {
                                            const int qb = requant_i8(double(yb[t1]) * sc * rq);
                                            *reinterpret_cast<uint16_t*>(d + rofs[t1]) = uint16_t((qa & 0xff) | ((qb & 0xff) << 8));
                                        } else {
                                            d[rofs[t1]] = int8_t(qa);
                                        }
                                    }
                                }
                            }
                            continue;
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
            __syncwarp();  // the warp has read its staged values
            if (lane == 0) ptx::mbar_arrive(&yempty[sb]);
#ifdef OM_TRACE
            if (et == 0) OM_STAMP(3, tu, 1);
            ++tu;
#endif
        }
    }
    __syncthreads();
#ifdef OM_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0 && units > 40 * int(gridDim.x)) {
        const long long t0 = s_trace[(0 * 32 + 8) * 4 + 0];
        for (int u2 = 8; u2 < 28; ++u2)
            printf("u%2d prod: free %6lld issued %6lld | mma: tempty %6lld full %6lld committed %6lld | A: tfull %6lld yempty %6lld staged %6lld | B: yfull %6lld stored %6lld\n",
                   u2, s_trace[(0 * 32 + u2) * 4 + 0] - t0, s_trace[(0 * 32 + u2) * 4 + 1] - t0,
                   s_trace[(1 * 32 + u2) * 4 + 0] - t0, s_trace[(1 * 32 + u2) * 4 + 1] - t0, s_trace[(1 * 32 + u2) * 4 + 2] - t0,
                   s_trace[(2 * 32 + u2) * 4 + 0] - t0, s_trace[(2 * 32 + u2) * 4 + 1] - t0, s_trace[(2 * 32 + u2) * 4 + 2] - t0,
                   s_trace[(3 * 32 + u2) * 4 + 0] - t0, s_trace[(3 * 32 + u2) * 4 + 1] - t0);
    }
#endif
    tl_mark(kTlOutput, 2);
    if (warp == kOmProdWarps) {
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
    OutPtrs od = o;
    if (const char* e = std::getenv("SFC_OM_DEBUG")) od.pairs |= std::atoi(e) << 8;
    return cudaLaunchKernelEx(&cfg, kern, tm, g, qp, sf, od, n_ob, n_tg, int(units), static_cast<const uint8_t*>(P));
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
