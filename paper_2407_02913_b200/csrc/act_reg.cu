// Register-resident activation transform for the 3x3 SFC variants (sfc4-4x4, sfc6-6x6,
// sfc6-7x7): V = B^T x B per (tile, channel) (gather_tiles, proj/src/quant.cpp:44-93), the
// PerTensor max|V| (quant.cpp:168-172) and the exact activation quantizer
// (quant.cpp:242-250).
//
// One CTA per (image, tile row, block of 2*PPW channels) covers the WHOLE tile row, so each
// channel's window rows are one contiguous byte band of NCHW: it is staged raw, 16 bytes per
// load (ld.global.nc.v4 of the 16-byte aligned chunks covering the band), into one shared
// plane per channel (odd word stride; even channels first so lanes stepping channel pairs
// hit distinct banks).  One thread then owns one tile and one channel pair (c, c+1) and
// builds its window in the two-lane SWAR form P = x'_c + 2^16 x'_{c+1} of the biased samples
// x' = x + 128 straight from the raw planes (three 32-bit shared loads + two funnel shifts per
// window row and channel, one LOP3 for the zero padding of quant.cpp:66-75 and the bias, one
// byte permute and a mask per sample pair).  The transforms are integer-linear and every
// intermediate stays in (-2^15, 2^15) (|V'| <= 9216), so one 32-bit add serves both channels;
// the bias adds 128 * rowsum_k * rowsum_l per lane to frequency (k, l) (the DC frequency only),
// removed together with the max/min lane bias in the horizontal pass.  The tile stays in registers: row
// transforms into n x K values, column transforms into V, each value consumed where formed:
//   MODE 0  max|V| only (unsigned 16x2 max/min of the biased words)
//   MODE 2  max|V| and the kept V (int16x2 words, V[f][t][c])
//   MODE 1  vq = q(V) with the verified quantizer of *vmax_in (two int8 per 16-bit store)
// Lane = channel pair (PPW pairs per warp); the rest of the lane index and the warp index
// select the tile column, so wide rows and narrow layers keep <= 10 warps per CTA.
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "devcache.hpp"
#include "sfc_kernels.hpp"
#include "sfc_tables.cuh"
#include "transforms.cuh"

namespace sfcb200 {

namespace {

constexpr int kRowMaxWarps = 10;  // CTA size bound: 320 threads

// The reference quantizer with clamping (the rare case without a verified multiply-shift):
// out of line, so the unrolled column loop stays small.
__device__ __noinline__ int quant_slow(int v, double sa, int qmax, unsigned long long* sat) {
    return clamp_q(exact_q(v, sa), qmax, sat);
}

// A 16-byte chunk that straddles an end of x: only its bytes inside [xlo, xhi), zeros elsewhere.
__device__ __noinline__ uint4 chunk_clipped(uintptr_t ad, uintptr_t xlo, uintptr_t xhi) {
    uint32_t w[4] = {0, 0, 0, 0};
    for (int e = 0; e < 16; ++e)
        if (ad + e >= xlo && ad + e < xhi)
            w[e >> 2] |= uint32_t(*reinterpret_cast<const uint8_t*>(ad + e)) << (8 * (e & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace

// Shared words per channel plane: a 4-word guard (window columns left of the band), the band
// (<= 15 bytes of chunk misalignment + n image rows) and a tail guard, rounded to odd.
template <int V>
__host__ __device__ inline int row_plane_words(int W) {
    const int w = 4 + (48 + Tab<V>::n * W + 3) / 4;
    return w | 1;
}
// RS: row pitch (words) for a chunk of tc tile columns: misalignment + window extent +
// funnel overrun; the plane holds n rows plus the guards, rounded to odd.
template <int V>
__host__ __device__ inline int row_seg_pitch(int tc) {
    return (15 + (tc - 1) * Tab<V>::M + Tab<V>::n + 12 + 3) / 4 + 1;
}
template <int V>
__host__ __device__ inline int row_seg_plane_words(int tc) {
    return (4 + Tab<V>::n * row_seg_pitch<V>(tc) + 4) | 1;
}

// RS = true (rows wider than kRowMaxWarps warps of tiles at 32 pairs per warp): a CTA covers a
// chunk of tc tile columns and stages one segment per (channel, window row) -- the columns
// its windows touch -- at row pitch rpw words inside the channel's plane; otherwise the CTA
// covers the whole tile row and each channel's band is one contiguous segment.
template <int V, int MODE, int PPW, bool RS>
__global__ void __launch_bounds__(32 * kRowMaxWarps, 2) k_act_row(const int8_t* __restrict__ x, ConvGeom g, int plw,
                                                              int rpw, int tc,
                                                              int* __restrict__ vmax, int16_t* __restrict__ vkeep,
                                                              const int* __restrict__ vmax_in, int bits,
                                                              QuantParams* __restrict__ qp_out,
                                                              int8_t* __restrict__ vqA,
                                                              unsigned long long* __restrict__ sat,
                                                              const QuantParams* __restrict__ qtab) {
    using T = Tab<V>;
    constexpr int n = T::n, K = T::K, M = T::M, TPW = 32 / PPW, NCH = 2 * PPW;
    constexpr int kTl = MODE == 1 ? kTlQuant : kTlAbsmax;
    // The window is transformed from the biased samples x + 128, so the transform of frequency
    // (k, l) carries 128 * rowsum_k * rowsum_l extra per lane (rowsum = the response of BT row k
    // to a constant; only the DC rows have one), removed in the horizontal pass.
    constexpr uint32_t kBias8 = 0x80808080u;
    auto in_corr = [](int k, int l) { return 128 * bt_rowsum<V>(k) * bt_rowsum<V>(l) * 0x10001; };
    extern __shared__ __align__(16) uint32_t s_raw[];
    tl_mark(kTl, 0);
    if (MODE != 1) griddep_launch_dependents();

    const int nchunk = RS ? (g.tw + tc - 1) / tc : 1;
    const int ti = RS ? blockIdx.x / nchunk : blockIdx.x, b = blockIdx.y, c0 = blockIdx.z * NCH;
    const int tj0 = RS ? (blockIdx.x - ti * nchunk) * tc : 0;
    const int ih0 = ti * M - g.pad;
    const int r_lo = max(ih0, 0), nr = min(ih0 + n, g.H) - r_lo;
    const size_t HW = size_t(g.H) * g.W;
    const int8_t* xb = x + (size_t(b) * g.C + c0) * HW + size_t(r_lo) * g.W;  // band of channel c0
    const uintptr_t xlo = reinterpret_cast<uintptr_t>(x), xhi = xlo + size_t(g.B) * g.C * HW;
    // staged columns [cs, ce): RS the chunk's windows, else whole rows
    const int cs = RS ? max(tj0 * M - g.pad, 0) : 0;
    const int ce = RS ? min((min(tj0 + tc, g.tw) - 1) * M - g.pad + n, g.W) : g.W;
    const int band = RS ? ce - cs : nr * g.W;  // bytes per segment
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    auto plane = [&](int ch) { return ((ch & 1) * PPW + (ch >> 1)) * plw + 4; };

    // ---- stage: per segment (a channel's band, or RS one (channel, row) piece), the 16-byte
    // chunks covering it.  The CTA's threads walk the flat (segment, chunk) index, so
    // consecutive lanes load consecutive chunks of a segment; kB chunks' loads are in flight
    // before any is stored.  Destinations are word offsets into s_raw (shared stores, no
    // generic pointers).
    {
        const int nchv = min(NCH, g.C - c0);
        const int nseg = RS ? nchv * nr : nchv;
        const int cq = (15 + band + 15) >> 4;  // chunk bound over every misalignment
        const int total = nseg * cq;
        const uintptr_t xb_u = reinterpret_cast<uintptr_t>(xb) + cs;
        // the CTA's chunks all lie inside x unless it holds the first or last bytes of x
        const bool inside = (xb_u & ~uintptr_t(15)) >= xlo &&
                            ((xb_u + size_t(nchv - 1) * HW + size_t(nr - 1) * g.W + band + 15) & ~uintptr_t(15)) <= xhi;
        constexpr int kB = 8;
        // idx / cq and sg / nr by multiply-high: umulhi(i, floor(2^32 / d) + 1) == i / d while
        // i * d < 2^32 (the magic's excess over 2^32 / d is below 1); d == 1 separately
        const bool cq_fast = cq > 1 && (unsigned long long)total * unsigned(cq) < (1ull << 32);
        const unsigned cq_mag = cq > 1 ? 0xffffffffu / unsigned(cq) + 1u : 0u;
        const unsigned nr_mag = (RS && nr > 1) ? 0xffffffffu / unsigned(nr) + 1u : 0u;
        const int nt = blockDim.x;
        for (int i0 = threadIdx.x; i0 < total; i0 += kB * nt) {
            uint4 v[kB];
            int dst[kB];
#pragma unroll
            for (int jj = 0; jj < kB; ++jj) {
                const int idx = i0 + jj * nt;
                const int sg = cq == 1 ? idx : (cq_fast ? int(__umulhi(unsigned(idx), cq_mag)) : idx / cq);
                const int q = idx - sg * cq;
                const int ch = RS ? (nr == 1 ? sg : int(__umulhi(unsigned(sg), nr_mag))) : sg;
                const int ir = RS ? sg - ch * nr : 0;
                const uintptr_t start = xb_u + size_t(ch) * HW + size_t(ir) * g.W;
                const int mis = int(start & 15);
                const uintptr_t ad = start - mis + 16 * q;
                dst[jj] = (idx < total && 16 * q < mis + band) ? plane(ch) + ir * rpw + 4 * q : -1;
                v[jj] = make_uint4(0, 0, 0, 0);
                if (dst[jj] < 0) continue;
                if (inside || (ad >= xlo && ad + 16 <= xhi)) {
                    v[jj] = __ldg(reinterpret_cast<const uint4*>(ad));
                } else {
                    v[jj] = chunk_clipped(ad, xlo, xhi);
                }
            }
#pragma unroll
            for (int jj = 0; jj < kB; ++jj)
                if (dst[jj] >= 0) {
                    uint32_t* d = s_raw + dst[jj];
                    d[0] = v[jj].x, d[1] = v[jj].y, d[2] = v[jj].z, d[3] = v[jj].w;
                }
        }
    }
    __syncthreads();

    const int p = lane % PPW, tj = tj0 + wid * TPW + lane / PPW;
    const int c = c0 + 2 * p;
    const bool active = tj < g.tw && c < g.C;
    const int t = (b * g.th + ti) * g.tw + tj;

    // ---- the window from the raw planes, SWAR-paired, zero padding by byte masks; then the
    // vertical pass y[k][s] = sum_r BT[k][r] x[r][s] (the horizontal pass below then forms
    // V[k][0..K) in frequency order f = k*K + l, so stores walk f with one pointer stride)
    int y[K][n];
    if (active) {
        int xw[n][n];
        const int wc0 = tj * M - g.pad;  // image column of window column 0
        // byte s of the window valid <=> 0 <= wc0 + s < W: bytes [slo, shi) of a 12-byte mask
        const int slo = max(0, -wc0), shi = min(n, g.W - wc0);
        uint32_t mk[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int lo = min(max(slo - 4 * j, 0), 4), hi = min(max(shi - 4 * j, 0), 4);
            mk[j] = (hi >= 4 ? 0xffffffffu : (1u << (8 * hi)) - 1u) & ~(lo >= 4 ? 0xffffffffu : (1u << (8 * lo)) - 1u);
        }
        const bool ok1 = c + 1 < g.C;
        const uint32_t* pe = s_raw + plane(2 * p);
        const uint32_t* po = s_raw + plane(2 * p + 1);
        // byte offset of window column 0 of window row ir in the plane: whole rows, the band's
        // 16-byte misalignment + ir * W + wc0; RS, ir * rpw words + the row piece's own
        // misalignment + (wc0 - cs)
        const uintptr_t ae = reinterpret_cast<uintptr_t>(xb + size_t(2 * p) * HW) + cs;
        const uintptr_t ao = reinterpret_cast<uintptr_t>(xb + size_t(2 * p + 1) * HW) + cs;
        const int me = int(ae & 15) + wc0 - cs, mo = int(ao & 15) + wc0 - cs;
        auto roff = [&](uintptr_t a, int m, int ir) {
            return RS ? ir * rpw * 4 + int((a + size_t(ir) * g.W) & 15) + (wc0 - cs) : m + ir * g.W;
        };
        constexpr int NW4 = (n + 3) / 4;  // window words per row
#pragma unroll
        for (int r = 0; r < n; ++r) {
            const int ir = ih0 + r - r_lo;  // row within the band
            uint32_t we[NW4], wo[NW4];
            if (ir >= 0 && ir < nr) {  // CTA-uniform
                // biased bytes x + 128 (x ^ 0x80), padding bytes 0x80 (x = 0): one LOP3
                auto row = [&](const uint32_t* pl, int off, uint32_t (&o)[NW4]) {
                    const int wi = off >> 2, sh = (off & 3) * 8;
                    uint32_t src[NW4 + 1];
#pragma unroll
                    for (int j = 0; j <= NW4; ++j) src[j] = pl[wi + j];
#pragma unroll
                    for (int j = 0; j < NW4; ++j) o[j] = (__funnelshift_r(src[j], src[j + 1], sh) & mk[j]) ^ kBias8;
                };
                row(pe, roff(ae, me, ir), we);
                row(po, roff(ao, mo, ir), wo);
                if (!ok1) {
#pragma unroll
                    for (int j = 0; j < NW4; ++j) wo[j] = kBias8;
                }
            } else {
#pragma unroll
                for (int j = 0; j < NW4; ++j) we[j] = wo[j] = kBias8;
            }
            // the biased samples are non-negative, so the SWAR word is the two bytes zero-
            // extended into the half-words: one byte permute and one mask per sample pair
#pragma unroll
            for (int s = 0; s < n; ++s) {
                switch (s & 3) {
                    case 0: xw[r][s] = int(__byte_perm(we[s >> 2], wo[s >> 2], 0x4400) & 0x00ff00ffu); break;
                    case 1: xw[r][s] = int(__byte_perm(we[s >> 2], wo[s >> 2], 0x5511) & 0x00ff00ffu); break;
                    case 2: xw[r][s] = int(__byte_perm(we[s >> 2], wo[s >> 2], 0x6622) & 0x00ff00ffu); break;
                    default: xw[r][s] = int(__byte_perm(we[s >> 2], wo[s >> 2], 0x7733) & 0x00ff00ffu); break;
                }
            }
        }
#pragma unroll
        for (int s = 0; s < n; ++s) {
            int col[n], yk[K];
#pragma unroll
            for (int r = 0; r < n; ++r) col[r] = xw[r][s];
            fwd1d<V>(col, yk);
#pragma unroll
            for (int k = 0; k < K; ++k) y[k][s] = yk[k];
        }
    }

    if constexpr (MODE == 1) {
        griddep_wait();  // the absmax pre-pass (and any multi-GPU MAX exchange) is complete
        tl_mark(kTl, 1);
        const QuantParams qp = qparams_for(*vmax_in, bits, qtab);  // (block-uniform call)
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) *qp_out = qp;
        griddep_launch_dependents();
        if (!active) return;
        // ---- columns, quantized: vq[f][t][c, c+1], one 16-bit store per pair
        const size_t fstride = size_t(g.Tpad) * g.Cpad / 2;  // 16-bit units between frequency planes
        int16_t* vq = reinterpret_cast<int16_t*>(vqA + size_t(t) * g.Cpad + c);
        // qlo(lo), qhi(v - lo): the high lane is quantized as hi * 2^16 (same quotient with the
        // multiplier's shift and rounding term scaled by 2^16), saving its unpack
        auto rows = [&](auto qlo, auto qhi) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                int v[K], cb[K];
#pragma unroll
                for (int l = 0; l < K; ++l) cb[l] = -in_corr(k, l);
                fwd1d_bias<V>(y[k], v, cb);
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    const int lo = int(int16_t(v[l]));
                    *vq = int16_t(__byte_perm(uint32_t(qlo(lo)), uint32_t(qhi(v[l] - lo)), 0x0040));
                    vq += fstride;  // f = k * K + l: next frequency plane
                }
            }
        };
        if (qp.exact && qp.shift >= 33) {
            // q = floor((v*mul + 2^(S-1)) / 2^S) = (hi32(v*mul) + 2^(S-33)) >> (S-32) for S >= 33
            // (the dropped low word only adds a fraction below one unit of the numerator):
            // one mad.hi and one shift; the high lane (hi * 2^16) with S + 16.
            const int mul = int(qp.mul), c = 1 << (qp.shift - 33), sh = qp.shift - 32;
            const int c16 = 1 << (qp.shift - 17), sh16 = qp.shift - 16;
            rows([=](int v) { return quant_hi32(v, mul, c, sh); }, [=](int v) { return quant_hi32(v, mul, c16, sh16); });
        } else if (qp.exact) {  // uniform over the grid: no per-value branch
            const int mul = int(qp.mul);
            const long long half = 1ll << (qp.shift - 1), half16 = half << 16;
            const int shift = qp.shift, shift16 = qp.shift + 16;
            rows([=](int v) { return quant_fast(v, mul, half, shift); },
                 [=](int v) { return quant_fast(v, mul, half16, shift16); });
        } else {
            const double sa = qp.sa;
            const int qmax = qp.qmax;
            rows([=](int v) { return quant_slow(v, sa, qmax, sat); },
                 [=](int v) { return quant_slow(v >> 16, sa, qmax, sat); });
        }
        tl_mark(kTl, 2);
    } else {
        // ---- horizontal pass: V[k][l] = sum_s BT[l][s] y[k][s]; max/min over the int16x2 words,
        // biased (+2^15 per lane) so unsigned 16x2 max/min order both lanes
        uint32_t mx = 0u, mn = 0xffffffffu;
        if (active) {
            const size_t fstride = size_t(g.Tpad) * g.Cpad / 2;  // words between frequency planes
            int* vk = MODE == 2 ? reinterpret_cast<int*>(vkeep + size_t(t) * g.Cpad + c) : nullptr;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                int v[K], cb[K];
#pragma unroll
                for (int l = 0; l < K; ++l) cb[l] = int(0x80008000u) - in_corr(k, l);
                fwd1d_bias<V>(y[k], v, cb);
                uint32_t u[K];
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    u[l] = uint32_t(v[l]);  // lane j -> V_j + 2^15 (mod 2^16)
                    if constexpr (MODE == 2) {
                        *vk = int(u[l] ^ 0x80008000u);
                        vk += fstride;  // f = k * K + l
                    }
                }
#pragma unroll
                for (int l = 0; l + 1 < K; l += 2) {  // three-input SIMD max/min
                    mx = __vimax3_u16x2(mx, u[l], u[l + 1]);
                    mn = __vimin3_u16x2(mn, u[l], u[l + 1]);
                }
                if constexpr (K % 2) {
                    mx = __vmaxu2(mx, u[K - 1]);
                    mn = __vminu2(mn, u[K - 1]);
                }
            }
        }
        int local = 0;
        if (active) {
            const int hi_max = int(mx >> 16) - 0x8000, lo_max = int(mx & 0xffff) - 0x8000;
            const int hi_min = int(mn >> 16) - 0x8000, lo_min = int(mn & 0xffff) - 0x8000;
            local = max(max(hi_max, lo_max), -min(hi_min, lo_min));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
        griddep_wait();  // under PDL: *vmax has been zeroed by the predecessor
        tl_mark(kTl, 1);
        if (lane == 0 && local > 0) atomicMax(vmax, local);
        tl_mark(kTl, 2);
    }
}

// ============================================================================ host
namespace {
// Pairs per warp: the largest of 32, 16, ... that is <= the layer's pairs (rounded up to a
// power of two) and keeps the whole tile row within kRowMaxWarps warps.
int row_ppw(const ConvGeom& g) {
    int ppw = 32;
    const int pairs = (g.C + 1) / 2;
    while (ppw > 1 && ppw / 2 >= pairs) ppw /= 2;
    while (ppw > 1 && (g.tw + 32 / ppw - 1) / (32 / ppw) > kRowMaxWarps) ppw /= 2;
    return ppw;
}

// Wide rows of wide layers (more tiles than kRowMaxWarps warps hold at 32 pairs, >= 64
// channels): row-chunk CTAs at 32 pairs per warp instead of narrowing the pairs per warp.
bool row_segmented(const ConvGeom& g) {
    const char* e = std::getenv("SFC_ACT_ROWSEG");  // "0": whole-row CTAs only (A/B knob)
    return !(e && e[0] == '0') && g.tw > kRowMaxWarps && g.C >= 64;
}

template <int V, int MODE, int PPW, bool RS = false>
cudaError_t row_launch(const int8_t* x, const ConvGeom& g, int* vmax, int16_t* vkeep, const int* vmax_in, int bits,
                       QuantParams* qp, int8_t* vqA, unsigned long long* sat, const QuantParams* qtab,
                       cudaStream_t st, bool pdl) {
    constexpr int TPW = 32 / PPW;
    // RS: chunks of kRowMaxWarps * TPW tile columns, balanced over the row
    const int nchunk = RS ? (g.tw + kRowMaxWarps * TPW - 1) / (kRowMaxWarps * TPW) : 1;
    const int tc = RS ? (g.tw + nchunk - 1) / nchunk : g.tw;
    const int nw = (tc + TPW - 1) / TPW;
    const int plw = RS ? row_seg_plane_words<V>(tc) : row_plane_words<V>(g.W);
    const int rpw = RS ? row_seg_pitch<V>(tc) : 0;
    const size_t smem = size_t(2 * PPW) * plw * 4;
    const long gz = (g.C + 2 * PPW - 1) / (2 * PPW);
    const long gx = long(g.th) * nchunk;
    if (nw > kRowMaxWarps || gx > 0x7fffffffL || g.B > 65535 || gz > 65535 || smem > 200 * 1024)
        return cudaErrorInvalidConfiguration;
    auto kern = k_act_row<V, MODE, PPW, RS>;
    static SmemOptIn opt_in;
    if (smem > 48 * 1024)
        if (cudaError_t e = opt_in.ensure(kern, smem); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(gx), unsigned(g.B), unsigned(gz));
    cfg.blockDim = dim3(32 * nw);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, x, g, plw, rpw, tc, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab);
}

template <int V, int MODE>
cudaError_t row_dispatch(const int8_t* x, const ConvGeom& g, int* vmax, int16_t* vkeep, const int* vmax_in, int bits,
                         QuantParams* qp, int8_t* vqA, unsigned long long* sat, const QuantParams* qtab,
                         cudaStream_t st, bool pdl) {
    if (row_segmented(g))
        return row_launch<V, MODE, 32, true>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);
    switch (row_ppw(g)) {
        case 32: return row_launch<V, MODE, 32>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);
        case 16: return row_launch<V, MODE, 16>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);
        case 8: return row_launch<V, MODE, 8>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);
        case 4: return row_launch<V, MODE, 4>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);
        case 2: return row_launch<V, MODE, 2>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);
        default: return row_launch<V, MODE, 1>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);
    }
}
}  // namespace

bool act_reg_wanted(int variant, const ConvGeom& g) {
    if (variant > 2 || g.pad > 8) return false;  // (the plane guards cover windows from column -8)
    const char* force = std::getenv("SFC_ACT_REG");  // "0": the shared-memory kernels (A/B knob)
    if (force && force[0] == '0') return false;
    if (row_segmented(g)) return true;
    const int ppw = row_ppw(g);
    const int nw = (g.tw + 32 / ppw - 1) / (32 / ppw);
    const size_t smem = size_t(2 * ppw) * (variant == 0   ? row_plane_words<0>(g.W)
                                           : variant == 1 ? row_plane_words<1>(g.W)
                                                          : row_plane_words<2>(g.W)) * 4;
    return nw <= kRowMaxWarps && smem <= 200 * 1024;
}

cudaError_t launch_act_reg(int variant, int mode, const int8_t* x, const ConvGeom& g, int* vmax, int16_t* vkeep,
                           const int* vmax_in, int bits, QuantParams* qp, int8_t* vqA, unsigned long long* sat,
                           cudaStream_t st, bool pdl) {
    const QuantParams* qtab = mode == 1 ? qparams_table(false) : nullptr;
#define SFC_ROW_MODES(VV)                                                                                         \
    if (mode == 1) return row_dispatch<VV, 1>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);     \
    if (vkeep) return row_dispatch<VV, 2>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);         \
    return row_dispatch<VV, 0>(x, g, vmax, vkeep, vmax_in, bits, qp, vqA, sat, qtab, st, pdl);
    switch (variant) {
        case 0: { SFC_ROW_MODES(0) }
        case 1: { SFC_ROW_MODES(1) }
        case 2: { SFC_ROW_MODES(2) }
        default: return cudaErrorInvalidValue;
    }
#undef SFC_ROW_MODES
}

SFC_TL_UNIT_READER(tl_read_reg)

}  // namespace sfcb200
