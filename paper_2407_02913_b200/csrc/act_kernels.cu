// Activation stage of the quantized SFC conv: V = B^T x B per (tile, channel),
// the global max|V| pre-pass, and exact quantization into the GEMM A operand.
// Reference: gather_tiles (proj/src/quant.cpp:44-93), the PerTensor activation
// scale (quant.cpp:168-172) and the activation quantize loop (quant.cpp:242-250).
//
// One CTA per (image b, tile row ti, chunk of CC channels) covers every tile
// column of that tile row.  Thread t owns channel c = t % CC and work-group
// j = t / CC.  The transform is separable and runs in shared-memory stages:
//   stage 0  the n window rows of each channel, copied word for word as they lie in NCHW
//   stage 1  Z[tj][r][l] = sum_s BT[l][s] x[r][tj*M + s]      items (tj, r), zero padding
//            (quant.cpp:66-75) applied here
//   stage 2  V[k][l]     = sum_r BT[k][r] Z[tj][r][l]         items (tj, l); MODE 1
//            quantizes and stores each value to its vq row (lanes = consecutive channels)
// Shared arrays are channel-innermost (or channel-strided with an odd word stride) so a
// warp touches distinct banks, and item decompositions divide by compile-time constants.
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "ptx.cuh"
#include "devcache.hpp"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"
#include "transforms.cuh"

namespace sfcb200 {

namespace {
constexpr int kActThreads = 256;

struct ActSmem {
    int nwp;      // 32-bit words per staged row piece (the piece's bytes from its 4-aligned start)
    int chw;      // words per staged channel: n * nwp, made odd so lanes stepping channels hit
                  // distinct banks
    size_t z_off, x_off, bytes;  // s_z first; s_x, then (once s_x is dead) the kept-V rows
};

// Shared-memory layout of one CTA covering `twc` tile columns of one tile row.
template <int V, int CC>
__host__ __device__ inline ActSmem act_smem(int W, int twc) {
    using T = Tab<V>;
    ActSmem s;
    const int pw = min((twc - 1) * T::M + T::n, W);  // widest row piece (window clipped to the image)
    s.nwp = (pw + 6) >> 2;
    s.chw = T::n * s.nwp;
    if ((s.chw & 1) == 0) s.chw += 1;
    s.z_off = 0;
    s.x_off = (size_t(twc) * T::n * T::K * CC * 2 + 15) & ~size_t(15);
    const size_t xb = size_t(s.chw) * 4 * CC, vb = size_t(twc) * T::F * CC * 2;
    s.bytes = s.x_off + (xb > vb ? xb : vb);
    return s;
}
}  // namespace

// MODE 0: max|V| -> atomicMax(*vmax); with vkeep != nullptr V itself is kept as int16
// vkeep[f][t][c] (row pitch Cpad) for the quantizer (streaming or inside the GEMM).
// MODE 1: quantize with the scale derived from *vmax_in and write vq[f][t][c] (row pitch
// Cpad) for f = k*K + l.
// Grid: x = tile row * column chunks + chunk (twc tile columns each), y = image, z =
// channel chunk of CC.  Shared memory is bounded by twc, so wide images keep CC = 32
// (64-byte kept-V rows) instead of narrowing the channel chunk.
template <int V, int MODE, int CC>
__global__ void __launch_bounds__(kActThreads) k_act(const int8_t* __restrict__ x, ConvGeom g, int twc,
                                                     int* __restrict__ vmax, const int* __restrict__ vmax_in, int bits,
                                                     QuantParams* __restrict__ qp_out, int8_t* __restrict__ vqA,
                                                     unsigned long long* __restrict__ sat,
                                                     const QuantParams* __restrict__ qtab, int16_t* __restrict__ vkeep) {
    using T = Tab<V>;
    constexpr int n = T::n, K = T::K, M = T::M;
    constexpr int TPC = kActThreads / CC;   // work-groups per channel
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr int kTl = MODE == 1 ? kTlQuant : kTlAbsmax;
    tl_mark(kTl, 0);
    if (MODE == 0) griddep_launch_dependents();

    const int W = g.W;
    const int nchunk = (g.tw + twc - 1) / twc;
    const int ti = blockIdx.x / nchunk, tj0 = (blockIdx.x - ti * nchunk) * twc;
    const int ntj = min(twc, g.tw - tj0);
    const int b = blockIdx.y, c0 = blockIdx.z * CC;
    const int nch = min(CC, g.C - c0);
    const ActSmem L = act_smem<V, CC>(W, twc);
    int8_t* s_x = reinterpret_cast<int8_t*>(smem + L.x_off);     // [CC][n][nwp words], channel stride chw
    int16_t* s_z = reinterpret_cast<int16_t*>(smem + L.z_off);   // [twc][n][K][CC]
    int16_t* s_v = reinterpret_cast<int16_t*>(smem + L.x_off);   // [twc][F][CC] kept V (after stage 1)
    const int c = threadIdx.x % CC, j = threadIdx.x / CC;

    // ---- stage 0: the window rows [r_lo, r_lo + nrows) x columns [cb_lo, cb_lo + pw) of each
    // channel, one row piece at a time, copied word for word from the piece's 4-byte-aligned
    // start (so a word lands where it lies: no byte scatter).  Zero padding is left to
    // stage 1.  Words past the end of x are assembled from bytes.  Offsets are 32-bit from
    // the CTA's first channel plane (CC planes span < 2^31 bytes).
    const int ih0 = ti * M - g.pad;
    const int r_lo = max(ih0, 0), nrows = min(ih0 + n, g.H) - r_lo;
    const int cb_lo = max(tj0 * M - g.pad, 0);
    const int pw = min((tj0 + ntj - 1) * M - g.pad + n, W) - cb_lo;
    const int HW = g.H * W;
    const int8_t* base = x + (size_t(b) * g.C + c0) * size_t(HW);
    const int bmis = int(reinterpret_cast<uintptr_t>(base) & 3);
    auto piece_off = [&](int ch, int r) { return ch * HW + (r_lo + r) * W + cb_lo; };  // from base
    {
        const long long avail64 = (long long)(size_t(g.B) * g.C * HW) - (long long)(base - x);
        const int avail = avail64 > 0x7fffffffll ? 0x7fffffff : int(avail64);
        const int nwp = L.nwp;
        const unsigned wmag = 0xffffffffu / unsigned(nwp) + 1u, rmag = 0xffffffffu / unsigned(nrows) + 1u;
        const int total = nch * nrows * nwp;
        constexpr int kJ = 4;
        for (int k0 = 0; k0 < total; k0 += kJ * kActThreads) {
            uint32_t v[kJ];
            int dst[kJ];
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj) {
                const int k = k0 + jj * kActThreads + int(threadIdx.x);
                const int cr = nwp == 1 ? k : int(__umulhi(unsigned(k), wmag)), w = k - cr * nwp;
                const int ch = nrows == 1 ? cr : int(__umulhi(unsigned(cr), rmag)), r = cr - ch * nrows;
                const int po = piece_off(ch, r);
                const int lo = 4 * w - ((bmis + po) & 3);  // piece index of the word's first byte
                const int a = po + lo;                     // its offset from base (4-aligned address)
                dst[jj] = (k < total && lo < pw) ? ch * L.chw + r * nwp + w : -1;
                v[jj] = 0;
                if (dst[jj] >= 0) {
                    if (a + 4 <= avail) {
                        v[jj] = __ldg(reinterpret_cast<const unsigned int*>(base + a));
                    } else {
                        for (int q = 0; q < 4 && a + q < avail; ++q) v[jj] |= uint32_t(uint8_t(__ldg(base + a + q))) << (8 * q);
                    }
                }
            }
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj)
                if (dst[jj] >= 0) reinterpret_cast<uint32_t*>(s_x)[dst[jj]] = v[jj];
        }
    }
    __syncthreads();

    // ---- stage 1: row transform, items (tj, r).  Rows outside the image and channels
    // beyond C are zero; columns outside [0, W) are zero (only border tiles test them).
    {
        const int8_t* cx = s_x + c * L.chw * 4;
        for (int idx = j; idx < ntj * n; idx += TPC) {
            const int r = idx % n, tjl = idx / n;
            const int ir = ih0 + r - r_lo;  // row within the staged window
            const int col0 = (tj0 + tjl) * M - g.pad;
            int xs[n];
            if (c >= nch || ir < 0 || ir >= nrows) {
#pragma unroll
                for (int s = 0; s < n; ++s) xs[s] = 0;
            } else {
                const int mis = (bmis + piece_off(c, ir)) & 3;
                const int8_t* src = cx + ir * L.nwp * 4 + mis + (col0 - cb_lo);
                if (col0 >= 0 && col0 + n <= W) {
#pragma unroll
                    for (int s = 0; s < n; ++s) xs[s] = src[s];
                } else {
#pragma unroll
                    for (int s = 0; s < n; ++s) xs[s] = unsigned(col0 + s) < unsigned(W) ? int(src[s]) : 0;
                }
            }
            int16_t* dst = s_z + ((tjl * n + r) * K) * CC + c;
            int z[K];
            fwd1d<V>(xs, z);
#pragma unroll
            for (int l = 0; l < K; ++l) dst[l * CC] = int16_t(z[l]);
        }
    }

    QuantParams qp{};
    if (MODE == 1) {
        griddep_wait();  // the absmax pre-pass (and any multi-GPU MAX exchange) is complete
        tl_mark(kTl, 1);
        qp = qparams_for(*vmax_in, bits, qtab);
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) *qp_out = qp;
    }
    __syncthreads();  // stage 1's s_z is complete (the table lookup does not synchronise)
    if (MODE == 1) griddep_launch_dependents();

    // ---- stage 2: column transform, items (tj, l); MODE 1 quantizes and stores each value
    // straight to its vq row (lanes = consecutive channels: CC contiguous bytes per store).
    const int t0 = (b * g.th + ti) * g.tw + tj0;  // the CTA's first tile
    int8_t* vrow = vqA + size_t(t0) * g.Cpad + c0 + c;
    const size_t fstride = size_t(g.Tpad) * g.Cpad, kstride = size_t(K) * fstride;
    int vhi = 0, vlo = 0;
    auto column = [&](auto quantize) {
        for (int idx = j; idx < ntj * K; idx += TPC) {
            const int l = idx % K, tj = idx / K;
            int zr[n];
#pragma unroll
            for (int r = 0; r < n; ++r) zr[r] = s_z[((tj * n + r) * K + l) * CC + c];
            int v[K];
            fwd1d<V>(zr, v);
            int8_t* p = vrow + size_t(l) * fstride + size_t(tj) * g.Cpad;  // f = l, then += K rows
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (MODE == 1) {
                    *p = int8_t(quantize(v[k]));
                    p += kstride;
                } else {
                    vhi = max(vhi, v[k]);
                    vlo = min(vlo, v[k]);
                    if (vkeep) s_v[(tj * T::F + k * K + l) * CC + c] = int16_t(v[k]);
                }
            }
        }
    };
    if (MODE != 1) {
        column([](int v) { return v; });
    } else if (qp.exact && qp.shift >= 33) {  // one mad.hi + shift per value (common.cuh)
        const int mul = int(qp.mul), c = 1 << (qp.shift - 33), sh = qp.shift - 32;
        column([=](int v) { return quant_hi32(v, mul, c, sh); });
    } else if (qp.exact) {  // uniform over the CTA: no per-value branch
        // mul < 2^31 (derive_qparams): one 32x32+64 -> 64 multiply-add and a funnel shift
        const int mul = int(qp.mul);
        const long long half = 1ll << (qp.shift - 1);
        const int shift = qp.shift;
        column([=](int v) { return quant_fast(v, mul, half, shift); });
    } else {
        column([&](int v) { return clamp_q(exact_q(v, qp.sa), qp.qmax, sat); });
    }

    if (MODE == 0 && vkeep) {
        // kept V rows (tj, f): CC int16 channels contiguous in shared memory and in
        // V[f][t][c0 .. c0+CC), moved in 16-byte (CC >= 8) or 8-byte (CC = 4) pieces
        __syncthreads();
        constexpr int kPB = CC >= 8 ? 16 : 8, kPR = CC * 2 / kPB;  // piece bytes, pieces per row
        for (int i = threadIdx.x; i < ntj * T::F * kPR; i += kActThreads) {
            const int pc = i % kPR, row = i / kPR;
            const int f = row % T::F, tj = row / T::F;
            const uint8_t* s = reinterpret_cast<const uint8_t*>(s_v + row * CC) + pc * kPB;
            uint8_t* d = reinterpret_cast<uint8_t*>(vkeep + (size_t(f) * g.Tpad + t0 + tj) * g.Cpad + c0) + pc * kPB;
            if (kPB == 16)
                *reinterpret_cast<uint4*>(d) = *reinterpret_cast<const uint4*>(s);
            else
                *reinterpret_cast<uint2*>(d) = *reinterpret_cast<const uint2*>(s);
        }
    }
    if (MODE == 0) {
        const int lane = threadIdx.x & 31;
        int local = max(vhi, -vlo);
#pragma unroll
        for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
        griddep_wait();  // under PDL: *vmax has been zeroed by the predecessor
        tl_mark(kTl, 1);
        if (lane == 0 && local > 0) atomicMax(vmax, local);
    }
    tl_mark(kTl, 2);
}

// ---------------------------------------------------------------------------------------
// Two-channel SWAR absmax / keep-V pass for the 3x3 variants (MODE 0 of k_act, reworked).
// One thread owns one tile and one adjacent channel pair (c, c+1), packed into one 32-bit
// register as P = x_c + 2^16 x_{c+1}.  The transforms are integer-linear and every value
// they form (window samples, row-transform Z, V) stays inside (-2^15, 2^15)
// (|V| <= 4608), so a 32-bit add of two packed values is the exact packed sum of both
// lanes: every addition of the scheduled transforms serves two channels.  The row
// transforms write Z to the warp's own shared-memory slab (lane-contiguous words:
// conflict-free, one word per channel pair), the column transforms read it back; both
// loops stay rolled so the code fits the instruction cache.  A V pair becomes its int16x2
// memory word (low lane's borrow undone: P + 2^16 [lane0 < 0]), is reduced with
// max/min.s16x2 and stored as one 32-bit word -- a warp (32 pairs = 64 channels of one
// tile) writes 128 contiguous bytes of the kept V row per frequency.
constexpr int kPairCC = 64;  // channels per CTA (one warp of pairs per tile)
constexpr int kPairMaxTiles = 4;

struct PairSmem {
    int nwp, chw;  // as ActSmem: words per staged row piece, words per staged channel (odd)
    size_t z_off, bytes;
};
template <int V>
__host__ __device__ inline PairSmem pair_smem(int W, int twc) {
    using T = Tab<V>;
    PairSmem s;
    const int pw = min((twc - 1) * T::M + T::n, W);
    s.nwp = (pw + 6) >> 2;
    s.chw = T::n * s.nwp;
    if ((s.chw & 1) == 0) s.chw += 1;
    s.z_off = (size_t(s.chw) * 4 * kPairCC + 15) & ~size_t(15);
    s.bytes = s.z_off + size_t(twc) * T::K * T::n * 32 * 4;
    return s;
}

// Grid: x = tile row * column chunks + chunk (twc tiles), y = image, z = 64-channel block;
// block = 32 * twc threads (warp w = tile column tj0 + w, lane = channel pair).
// MODE 0: max|V| (+ kept V when vkeep); MODE 1: quantize with the scale of *vmax_in and write
// vq[f][t][c] (both channels of a pair as one 16-bit store: 64 contiguous bytes per warp).
template <int V, int MODE>
__global__ void __launch_bounds__(32 * kPairMaxTiles)
    k_act_pair(const int8_t* __restrict__ x, ConvGeom g, int twc, int* __restrict__ vmax, int16_t* __restrict__ vkeep,
               const int* __restrict__ vmax_in, int bits, QuantParams* __restrict__ qp_out,
               int8_t* __restrict__ vqA, unsigned long long* __restrict__ sat, const QuantParams* __restrict__ qtab) {
    using T = Tab<V>;
    constexpr int n = T::n, K = T::K, M = T::M;
    constexpr int kTl = MODE == 1 ? kTlQuant : kTlAbsmax;
    extern __shared__ __align__(16) uint8_t smem[];
    tl_mark(kTl, 0);
    if (MODE == 0) griddep_launch_dependents();

    const int W = g.W;
    const int nchunk = (g.tw + twc - 1) / twc;
    const int ti = blockIdx.x / nchunk, tj0 = (blockIdx.x - ti * nchunk) * twc;
    const int ntj = min(twc, g.tw - tj0);
    const int b = blockIdx.y, c0 = blockIdx.z * kPairCC;
    const int nch = min(kPairCC, g.C - c0);
    const PairSmem L = pair_smem<V>(W, twc);
    uint32_t* s_xw = reinterpret_cast<uint32_t*>(smem);
    // staged plane of channel ch: even channels first, then odd ones, so lane p's two loads
    // (channels 2p, 2p+1) step through planes with the odd word stride chw: no bank conflicts
    auto plane = [&](int ch) { return ((ch & 1) * (kPairCC / 2) + (ch >> 1)) * L.chw; };

    // ---- stage 0: window rows [r_lo, r_lo + nrows) x columns [cb_lo, cb_lo + pw) of each
    // channel; word w of a staged row holds columns cb_lo + 4w .. +3 (funnel-shifted from the
    // two aligned words that cover them), so a sample's shared address needs no per-row
    // alignment term.  Words past the end of x read as zero.
    const int ih0 = ti * M - g.pad;
    const int r_lo = max(ih0, 0), nrows = min(ih0 + n, g.H) - r_lo;
    const int cb_lo = max(tj0 * M - g.pad, 0);
    const int pw = min((tj0 + ntj - 1) * M - g.pad + n, W) - cb_lo;
    const int HW = g.H * W;
    const int8_t* base = x + (size_t(b) * g.C + c0) * size_t(HW);
    {
        const uint32_t* xw = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(base) & ~uintptr_t(3));
        const int bmis = int(reinterpret_cast<uintptr_t>(base) & 3);
        const long long availw64 = ((long long)(size_t(g.B) * g.C * HW) - (long long)(base - x) + bmis + 3) >> 2;
        const int availw = availw64 > 0x7fffffffll ? 0x7fffffff : int(availw64);  // readable words from xw
        const int nwp = (pw + 3) >> 2;
        const unsigned wmag = 0xffffffffu / unsigned(nwp) + 1u, rmag = 0xffffffffu / unsigned(nrows) + 1u;
        const int total = nch * nrows * nwp;
        constexpr int kJ = 8;  // loads in flight per thread
        for (int k0 = 0; k0 < total; k0 += kJ * int(blockDim.x)) {
            uint32_t lo[kJ], hi[kJ];
            int dst[kJ], sh[kJ];
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj) {
                const int k = k0 + jj * int(blockDim.x) + int(threadIdx.x);
                const int cr = nwp == 1 ? k : int(__umulhi(unsigned(k), wmag)), w = k - cr * nwp;
                const int ch = nrows == 1 ? cr : int(__umulhi(unsigned(cr), rmag)), r = cr - ch * nrows;
                const int byte = bmis + ch * HW + (r_lo + r) * W + cb_lo + 4 * w;  // from xw
                const int a = byte >> 2;
                sh[jj] = (byte & 3) * 8;
                dst[jj] = k < total ? plane(ch) + r * L.nwp + w : -1;
                lo[jj] = (dst[jj] >= 0 && a < availw) ? __ldg(xw + a) : 0u;
                hi[jj] = (dst[jj] >= 0 && sh[jj] && a + 1 < availw) ? __ldg(xw + a + 1) : 0u;
            }
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj)
                if (dst[jj] >= 0) s_xw[dst[jj]] = __funnelshift_r(lo[jj], hi[jj], sh[jj]);
        }
    }
    __syncthreads();

    const int tjl = threadIdx.x >> 5, p = threadIdx.x & 31, c = 2 * p;
    int mx = 0, mn = 0;  // int16x2 running max / min of V over this thread's two channels
    int* sz = reinterpret_cast<int*>(smem + L.z_off) + tjl * (K * n * 32) + p;  // [l][r][lane]
    if (tjl < ntj) {
        const int col0 = (tj0 + tjl) * M - g.pad;
        // interior tile with both channels present: no per-sample predicates
        const bool fast = col0 >= 0 && col0 + n <= W && c + 1 < nch;
        const int8_t* px0 = reinterpret_cast<const int8_t*>(s_xw + plane(c)) + (col0 - cb_lo);
        const int8_t* px1 = reinterpret_cast<const int8_t*>(s_xw + plane(c + 1)) + (col0 - cb_lo);
        const bool ok0 = c < nch, ok1 = c + 1 < nch;
        // ---- rows: Z[r][l] = sum_s BT[l][s] x[r][s], both channels at once
#pragma unroll 1
        for (int r = 0; r < n; ++r) {
            const int ir = ih0 + r - r_lo;  // row within the staged window
            int xs[n], z[K];
            if (ir < 0 || ir >= nrows) {
#pragma unroll
                for (int s2 = 0; s2 < n; ++s2) xs[s2] = 0;
            } else if (fast) {
                const int8_t* s0 = px0 + ir * L.nwp * 4;
                const int8_t* s1 = px1 + ir * L.nwp * 4;
#pragma unroll
                for (int s2 = 0; s2 < n; ++s2) xs[s2] = int(s0[s2]) + (int(s1[s2]) << 16);
            } else {
                const int8_t* s0 = px0 + ir * L.nwp * 4;
                const int8_t* s1 = px1 + ir * L.nwp * 4;
#pragma unroll
                for (int s2 = 0; s2 < n; ++s2) {
                    const bool in = unsigned(col0 + s2) < unsigned(W);
                    const int a = (ok0 && in) ? int(s0[s2]) : 0;
                    const int h = (ok1 && in) ? int(s1[s2]) : 0;
                    xs[s2] = a + (h << 16);
                }
            }
            fwd1d<V>(xs, z);
#pragma unroll
            for (int l = 0; l < K; ++l) sz[(l * n + r) * 32] = z[l];
        }
    }
    QuantParams qp{};
    if (MODE == 1) {  // every thread: the table fallback derives cooperatively over the block
        griddep_wait();  // the absmax pre-pass (and any multi-GPU MAX exchange) is complete
        tl_mark(kTl, 1);
        qp = qparams_for(*vmax_in, bits, qtab);
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) *qp_out = qp;
        griddep_launch_dependents();
    }
    __syncwarp();
    if (MODE == 1 && tjl < ntj) {
        // ---- columns, quantized: vq[f][t][c, c+1] (one 16-bit store per pair)
        const int t = (b * g.th + ti) * g.tw + tj0 + tjl;
        const size_t fstride = size_t(g.Tpad) * g.Cpad / 2;  // 16-bit units between frequency planes
        int16_t* vq = reinterpret_cast<int16_t*>(vqA + size_t(t) * g.Cpad + c0 + c);
        auto columns = [&](auto quantize) {
#pragma unroll 1
            for (int l = 0; l < K; ++l) {
                int zr[n], v[K];
#pragma unroll
                for (int r = 0; r < n; ++r) zr[r] = sz[(l * n + r) * 32];
                fwd1d<V>(zr, v);
                int16_t* q = vq;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int lo = int(int16_t(v[k])), hi = (v[k] - lo) >> 16;  // unpack the pair
                    *q = int16_t((quantize(lo) & 0xff) | (quantize(hi) << 8));
                    q += K * fstride;  // f = k * K + l: next k
                }
                vq += fstride;  // next l
            }
        };
        if (qp.exact && qp.shift >= 33) {  // one mad.hi + shift per value (common.cuh)
            const int mul = int(qp.mul), c = 1 << (qp.shift - 33), sh = qp.shift - 32;
            columns([=](int v) { return quant_hi32(v, mul, c, sh); });
        } else if (qp.exact) {  // uniform over the grid: no per-value branch
            const int mul = int(qp.mul);
            const long long half = 1ll << (qp.shift - 1);
            const int shift = qp.shift;
            columns([=](int v) { return quant_fast(v, mul, half, shift); });
        } else {
            columns([&](int v) { return clamp_q(exact_q(v, qp.sa), qp.qmax, sat); });
        }
    }
    if (MODE == 0 && tjl < ntj) {
        // ---- columns: V[k][l] = sum_r BT[k][r] Z[r][l]; keep as int16x2 words
        const int t = (b * g.th + ti) * g.tw + tj0 + tjl;
        const size_t fstride = size_t(g.Tpad) * g.Cpad / 2;  // words between frequency planes
        int* vk = vkeep ? reinterpret_cast<int*>(vkeep + size_t(t) * g.Cpad + c0 + c) : nullptr;
#pragma unroll 1
        for (int l = 0; l < K; ++l) {
            int zr[n], v[K];
#pragma unroll
            for (int r = 0; r < n; ++r) zr[r] = sz[(l * n + r) * 32];
            fwd1d<V>(zr, v);
            int* q = vk;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int w = v[k] + ((v[k] & 0x8000) << 1);  // P -> int16x2 word
                mx = __vmaxs2(mx, w);
                mn = __vmins2(mn, w);
                if (vk) {
                    *q = w;
                    q += K * fstride;  // f = k * K + l: next k
                }
            }
            if (vk) vk += fstride;  // next l
        }
    }
    if (MODE == 0) {
        int local = max(max(int(int16_t(mx)), mx >> 16), -min(int(int16_t(mn)), mn >> 16));
#pragma unroll
        for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
        griddep_wait();  // under PDL: *vmax has been zeroed by the predecessor
        tl_mark(kTl, 1);
        if (p == 0 && local > 0) atomicMax(vmax, local);
    }
    tl_mark(kTl, 2);
}

// Streaming quantizer over the V kept by the absmax pass: vq[f][t][c] = q(V[f][t][c]) for
// t < T, 16 channels per item (two 16-byte loads, one 16-byte store); channels >= C are
// written as 0.  HBM-bound: 3 bytes per value.
__global__ void __launch_bounds__(kActThreads) k_quant_kept(const int16_t* __restrict__ vkeep, ConvGeom g, int F,
                                                            const int* __restrict__ vmax_in, int bits,
                                                            QuantParams* __restrict__ qp_out,
                                                            int8_t* __restrict__ vqA,
                                                            unsigned long long* __restrict__ sat,
                                                            const QuantParams* __restrict__ qtab) {
    tl_mark(kTlQuant, 0);
    griddep_wait();  // V and the (all-reduced) vmax are complete
    tl_mark(kTlQuant, 1);
    const QuantParams qp = qparams_for(*vmax_in, bits, qtab);
    if (threadIdx.x == 0 && blockIdx.x == 0) *qp_out = qp;
    griddep_launch_dependents();
    // grid = (x blocks striding over the (t, chunk) items of one frequency, F)
    const int chunks = g.Cpad / 16;
    const unsigned items = unsigned(g.T) * unsigned(chunks);  // < 2^32 / chunks (host check)
    const unsigned cmagic = 0xffffffffu / unsigned(chunks) + 1u;
    const size_t fbase = size_t(blockIdx.y) * g.Tpad * g.Cpad;
    // kU items per thread per round: all their loads are in flight before the first is used.
    constexpr int kU = 4;
    const unsigned stride = gridDim.x * blockDim.x;
    auto run = [&](auto quantize) {
        for (unsigned it0 = blockIdx.x * blockDim.x + threadIdx.x; it0 < items; it0 += kU * stride) {
            uint4 a[kU], b[kU];
            size_t off[kU];
            int cb[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const unsigned it = it0 + u * stride;
                const unsigned t = chunks == 1 ? it : __umulhi(it, cmagic);
                const int q = int(it - t * unsigned(chunks));
                off[u] = fbase + size_t(t) * g.Cpad + size_t(q) * 16;
                cb[u] = it < items ? q * 16 : 1 << 30;  // (out of range: no load, no store)
                a[u] = b[u] = make_uint4(0, 0, 0, 0);
                if (cb[u] < g.C) {
                    const uint4* src = reinterpret_cast<const uint4*>(vkeep + off[u]);
                    a[u] = __ldcs(src);  // streamed once
                    b[u] = __ldcs(src + 1);
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
            if (cb[u] == (1 << 30)) continue;
            uint4 out = make_uint4(0, 0, 0, 0);
            const int cbase = cb[u];
            if (cbase < g.C) {
                uint32_t w[8] = {a[u].x, a[u].y, a[u].z, a[u].w, b[u].x, b[u].y, b[u].z, b[u].w};
                if (cbase + 16 > g.C) {  // channels >= C of the tail chunk: V there is not defined
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (cbase + e >= g.C) w[e >> 1] &= ~(0xffffu << (16 * (e & 1)));
                }
                uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
                for (int e = 0; e < 16; ++e) {  // (quantize(0) == 0: no saturation from padding)
                    const int v = int(int16_t(w[e >> 1] >> (16 * (e & 1))));
                    o[e >> 2] |= uint32_t(uint8_t(int8_t(quantize(v)))) << (8 * (e & 3));
                }
                out = make_uint4(o[0], o[1], o[2], o[3]);
            }
            *reinterpret_cast<uint4*>(vqA + off[u]) = out;
            }
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
    } else {
        run([&](int v) { return clamp_q(exact_q(v, qp.sa), qp.qmax, sat); });
    }
    tl_mark(kTlQuant, 2);
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

template <int V, int MODE, int CC>
cudaError_t act_launch_cc(const int8_t* x, const ConvGeom& g, int twc, int* vmax, const int* vmax_in, int bits,
                          QuantParams* qp, int8_t* vqA, unsigned long long* sat, int16_t* vkeep, cudaStream_t st,
                          bool pdl) {
    const size_t smem = act_smem<V, CC>(g.W, twc).bytes;
    auto kern = k_act<V, MODE, CC>;
    static SmemOptIn opt_in;  // per instantiation and device: raised only when a layer needs more
    if (cudaError_t e = opt_in.ensure(kern, smem); e != cudaSuccess) return e;
    const long gx = long(g.th) * ((g.tw + twc - 1) / twc);
    if (gx > 0x7fffffffL || g.B > 65535 || (g.C + CC - 1) / CC > 65535) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(gx), g.B, (g.C + CC - 1) / CC);
    cfg.blockDim = dim3(kActThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, x, g, twc, vmax, vmax_in, bits, qp, vqA, sat,
                              MODE == 0 ? nullptr : qparams_table(false), vkeep);
}

// CTA shape: CC = 32 channels (64-byte kept-V rows, 32-byte vq rows) unless the layer has
// fewer channels; tile columns per CTA (twc) halved until shared memory is <= 64 KB and the
// grid has two waves over the 148 SMs; only then narrower channel chunks.
template <int V>
void pick_shape(const ConvGeom& g, int& cc, int& twc) {
    cc = 32;
    while (cc > 4 && cc / 2 >= g.C) cc /= 2;
    twc = g.tw;
    auto bytes = [&](int c, int t) {
        return c == 32 ? act_smem<V, 32>(g.W, t).bytes
             : c == 16 ? act_smem<V, 16>(g.W, t).bytes
             : c == 8  ? act_smem<V, 8>(g.W, t).bytes
                       : act_smem<V, 4>(g.W, t).bytes;
    };
    auto ctas = [&](int c, int t) { return long(g.th) * ((g.tw + t - 1) / t) * g.B * ((g.C + c - 1) / c); };
    while (twc > 1 && bytes(cc, twc) > 64 * 1024) twc = (twc + 1) / 2;
    while (twc > 1 && ctas(cc, twc) < 2 * 148) twc = (twc + 1) / 2;
    while (cc > 4 && ctas(cc, twc) < 2 * 148) cc /= 2;
    while (cc > 4 && bytes(cc, twc) > 96 * 1024) cc /= 2;
}

}  // namespace

bool act_pair_wanted(const ConvGeom& g) {
    const char* force = std::getenv("SFC_ACT_PAIR");  // "0" / "1": A/B measurement / test knob
    return force ? force[0] == '1' : long(g.T) * ((g.C + 1) / 2) >= 32768;
}

namespace {
// k_act_pair: tiles per CTA halved until the grid has two waves over the 148 SMs.
template <int V, int MODE>
cudaError_t act_pair_launch(const int8_t* x, const ConvGeom& g, int* vmax, const int* vmax_in, int bits,
                            QuantParams* qp, int8_t* vqA, unsigned long long* sat, int16_t* vkeep, cudaStream_t st,
                            bool pdl) {
    int twc = g.tw < kPairMaxTiles ? g.tw : kPairMaxTiles;
    const long blocks_c = (g.C + kPairCC - 1) / kPairCC;
    auto ctas = [&](int t) { return long(g.th) * ((g.tw + t - 1) / t) * g.B * blocks_c; };
    while (twc > 1 && ctas(twc) < 2 * 148) twc = (twc + 1) / 2;
    const size_t smem = pair_smem<V>(g.W, twc).bytes;
    auto kern = k_act_pair<V, MODE>;
    static SmemOptIn opt_in;
    if (cudaError_t e = opt_in.ensure(kern, smem); e != cudaSuccess) return e;
    const long gx = long(g.th) * ((g.tw + twc - 1) / twc);
    if (gx > 0x7fffffffL || g.B > 65535 || blocks_c > 65535) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(gx), g.B, unsigned(blocks_c));
    cfg.blockDim = dim3(32 * twc);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, x, g, twc, vmax, vkeep, vmax_in, bits, qp, vqA, sat,
                              MODE == 0 ? nullptr : qparams_table(false));
}

template <int V, int MODE>
cudaError_t act_launch(const int8_t* x, const ConvGeom& g, int* vmax, const int* vmax_in, int bits, QuantParams* qp,
                       int8_t* vqA, unsigned long long* sat, int16_t* vkeep, cudaStream_t st, bool pdl) {
    if (act_reg_wanted(V, g))
        return launch_act_reg(V, MODE, x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, st, pdl);
    if constexpr (V <= 2) {
        // the SWAR kernel has one thread per (tile, channel pair): it needs >= 32k of them to
        // fill the GPU (measured: config 5 absmax 0.121 -> 0.091 ms, ResNet-18 layers 0.435 ->
        // 0.382 ms); smaller layers (config 2) keep the item-parallel kernel
        if (act_pair_wanted(g))
            return act_pair_launch<V, MODE>(x, g, vmax, vmax_in, bits, qp, vqA, sat, vkeep, st, pdl);
    }
    int cc, twc;
    pick_shape<V>(g, cc, twc);
    switch (cc) {
        case 32: return act_launch_cc<V, MODE, 32>(x, g, twc, vmax, vmax_in, bits, qp, vqA, sat, vkeep, st, pdl);
        case 16: return act_launch_cc<V, MODE, 16>(x, g, twc, vmax, vmax_in, bits, qp, vqA, sat, vkeep, st, pdl);
        case 8: return act_launch_cc<V, MODE, 8>(x, g, twc, vmax, vmax_in, bits, qp, vqA, sat, vkeep, st, pdl);
        default: return act_launch_cc<V, MODE, 4>(x, g, twc, vmax, vmax_in, bits, qp, vqA, sat, vkeep, st, pdl);
    }
}

}  // namespace

cudaError_t launch_act_absmax(int variant, const int8_t* x, const ConvGeom& g, int* vmax, int16_t* vkeep,
                              cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return act_launch<0, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, vkeep, st, pdl);
        case 1: return act_launch<1, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, vkeep, st, pdl);
        case 2: return act_launch<2, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, vkeep, st, pdl);
        case 3: return act_launch<3, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, vkeep, st, pdl);
        default: return act_launch<4, 0>(x, g, vmax, nullptr, 8, nullptr, nullptr, nullptr, vkeep, st, pdl);
    }
}

cudaError_t launch_act_quant(int variant, const int8_t* x, const ConvGeom& g, const int* vmax, int bits,
                             QuantParams* qp, int8_t* vqA, unsigned long long* sat, cudaStream_t st, bool pdl) {
    switch (variant) {
        case 0: return act_launch<0, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, nullptr, st, pdl);
        case 1: return act_launch<1, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, nullptr, st, pdl);
        case 2: return act_launch<2, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, nullptr, st, pdl);
        case 3: return act_launch<3, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, nullptr, st, pdl);
        default: return act_launch<4, 1>(x, g, nullptr, vmax, bits, qp, vqA, sat, nullptr, st, pdl);
    }
}

cudaError_t launch_quant_kept(const int16_t* vkeep, const ConvGeom& g, int F, const int* vmax, int bits,
                              QuantParams* qp, int8_t* vqA, unsigned long long* sat, cudaStream_t st, bool pdl) {
    const long items = long(g.T) * (g.Cpad / 16);
    if (items * (g.Cpad / 16) >= (1l << 32)) return cudaErrorInvalidValue;
    const long want = (items + kActThreads - 1) / kActThreads, cap = (148L * 8 + F - 1) / F;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(want < cap ? want : cap), unsigned(F));
    cfg.blockDim = dim3(kActThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_quant_kept, vkeep, g, F, vmax, bits, qp, vqA, sat, qparams_table(false));
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
