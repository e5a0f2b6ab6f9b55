// Device helpers shared by the SFC kernels: exact activation quantizer and
// programmatic-dependent-launch (PDL) controls.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "sfc_kernels.hpp"

namespace sfcb200 {

constexpr int kRowsPerTile = 128;  // GEMM M block (tiles per CTA)

// ---------------------------------------------------------------- PDL
// A kernel launched with programmatic stream serialization may start while its
// predecessor is still running; everything before griddep_wait() overlaps the
// predecessor's tail, everything after sees its results.  Both are no-ops for
// kernels launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- timeline (debug build)
// Built with -DSFC_TIMELINE (make TIMELINE=1 -> libsfc_b200_tl.so): thread 0 of every CTA
// stamps %globaltimer at kernel entry (slot 0, min over CTAs), after its dependency wait
// (slot 1, min) and at exit (slot 2, max), per kernel id; sfc_debug_timeline() reads them.
#ifdef SFC_TIMELINE
static __device__ unsigned long long g_tl[kTlCount][3];
__device__ __forceinline__ void tl_mark(int id, int which) {
    if (threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (which == 2)
        atomicMax(&g_tl[id][2], t);
    else
        atomicMin(&g_tl[id][which], t);
}
// Per translation unit: copy out (and re-arm) this unit's stamps, merged by the caller.
#define SFC_TL_UNIT_READER(fn)                                                                  \
    cudaError_t fn(unsigned long long* out, bool reset) {                                     \
        cudaError_t e = cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl));                         \
        if (e != cudaSuccess || !reset) return e;                                              \
        unsigned long long init[kTlCount][3];                                                  \
        for (int i = 0; i < kTlCount; ++i) init[i][0] = init[i][1] = ~0ull, init[i][2] = 0ull; \
        return cudaMemcpyToSymbol(g_tl, init, sizeof(init));                                   \
    }
#else
__device__ __forceinline__ void tl_mark(int, int) {}
#define SFC_TL_UNIT_READER(fn) \
    cudaError_t fn(unsigned long long*, bool) { return cudaErrorNotSupported; }
#endif

// ---------------------------------------------------------------- quantization
__device__ __forceinline__ int clamp_q(int q, int qmax, unsigned long long* sat) {
    const int qmin = -qmax - 1;
    if (q > qmax || q < qmin) {
        atomicAdd(sat, 1ull);
        q = q > qmax ? qmax : qmin;
    }
    return q;
}

// The reference quantizer: nearbyint(double(v) / scale) (quant.cpp:102-115).
__device__ __forceinline__ int exact_q(long long v, double sa) { return int(rint(__ddiv_rn(double(v), sa))); }

// The verified multiply-shift quantizer: (v * mul + half) >> shift with mul < 2^31, as one
// mad.wide.s32 (IMAD.WIDE with the 64-bit rounding addend) and one funnel shift.
__device__ __forceinline__ int quant_fast(int v, int mul, long long half, int shift) {
    long long r;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(v), "r"(mul), "l"(half));
    return int(r >> shift);
}

// The same quotient for S >= 33: floor((v*mul + 2^(S-1)) / 2^S) = (hi32(v*mul) + 2^(S-33)) >>
// (S-32) -- the dropped low word only adds a fraction below one unit of the numerator -- as one
// mad.hi.s32 and one shift (c = 2^(S-33), sh = S-32).
__device__ __forceinline__ int quant_hi32(int v, int mul, int c, int sh) {
    int r;
    asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "r"(mul), "r"(c));
    return r >> sh;
}

// Activation quantizer.  Fast path (qp.exact): one 32x32->64 multiply-add and a
// shift, proven equal to exact_q for every |v| <= vmax by derive_qparams (so no
// clamp can trigger).  Otherwise the per-element fp64 division with clamping.
__device__ __forceinline__ int quant_act(int v, const QuantParams& qp, unsigned long long* sat) {
    if (qp.exact) return quant_fast(v, int(qp.mul), 1ll << (qp.shift - 1), qp.shift);
    return clamp_q(exact_q(v, qp.sa), qp.qmax, sat);
}

__device__ __forceinline__ long long qcand(long long m0, int c) {
    return m0 + (c == 0 ? 0 : ((c & 1) ? (c + 1) / 2 : -(c / 2)));
}

// sa = max(vmax / qmax, 1e-8) (scale_minmax, quant.cpp:117-120) and a verified
// multiply-shift quantizer, computed by ONE warp.
//
// fast(v) = floor((v * mul + 2^(S-1)) / 2^S) and exact(v) = rint(fl(v / sa)) are
// both monotone non-decreasing step functions of the integer v with value 0 at
// v = 0, so they agree on [-vmax, vmax] iff their level crossings agree.  For each
// level k = 0..qmax the fast crossing on the positive side is
// v_k = ceil((2k+1) 2^(S-1) / mul) and on the negative side
// w_k = floor((2k+1) 2^(S-1) / mul) + 1; checking exact() on both sides of each
// crossing (or exact(vmax) <= k when the crossing lies beyond vmax) proves
// equality over the whole range with ~4 (qmax+1) fp64 divisions instead of
// 2 vmax + 1.  Including k = qmax proves |fast(v)| <= qmax, i.e. no clamping.
__device__ __forceinline__ bool qlevel_bad(int k, int vmax, double sa, long long mul, int S) {
    const long long num = (long long)(2 * k + 1) << (S - 1);
    const long long vk = (num + mul - 1) / mul;
    const long long wk = num / mul + 1;
    bool bad = false;
    if (vk <= vmax)
        bad |= exact_q(vk, sa) < k + 1 || exact_q(vk - 1, sa) > k;
    else
        bad |= exact_q(vmax, sa) > k;
    if (wk <= vmax)
        bad |= exact_q(wk, sa) < k + 1 || exact_q(wk - 1, sa) > k;
    else
        bad |= exact_q(vmax, sa) > k;
    return bad;
}

// Block-cooperative variant: every thread of the CTA must call it (uses
// __syncthreads_or); one level per thread for 8-bit and 256+ threads.
__device__ __forceinline__ QuantParams derive_qparams_block(int vmax, int bits) {
    const int qmax = (1 << (bits - 1)) - 1;
    const double sa = fmax(double(vmax) / double(qmax), 1e-8);
    int e;
    frexp(sa, &e);
    const int S = 29 + e;
    const long long m0 = (long long)floor(ldexp(1.0, S) / sa);
    int found = -1;
    for (int cand = 0; cand < 5; ++cand) {
        const long long mul = qcand(m0, cand);
        bool bad = mul <= 0;
        for (int k = threadIdx.x; k <= qmax && !bad; k += blockDim.x) bad = qlevel_bad(k, vmax, sa, mul, S);
        if (!__syncthreads_or(bad)) {
            found = cand;
            break;
        }
    }
    QuantParams p;
    p.sa = sa;
    p.shift = S;
    p.vmax = vmax;
    p.qmax = qmax;
    p.exact = found >= 0;
    p.mul = qcand(m0, found >= 0 ? found : 0);
    return p;
}

// Quantizer parameters for every (bits, vmax) with bits in [2, 8] and vmax <= 4608 (the
// largest |V| any catalogued algorithm produces from int8 inputs: (max row L1 of B^T)^2 * 128
// = 6^2 * 128), derived once per device (build_qparams_table) so a CTA pays one dependent
// load instead of the derivation; other vmax fall back to derive_qparams_block.
constexpr int kQpTableMax = 4608;
constexpr int kQpTableEntries = 7 * (kQpTableMax + 1);
// Block-uniform; every thread of the CTA must call it (the fallback synchronises).
__device__ __forceinline__ QuantParams derive_qparams_block(int vmax, int bits);
__device__ __forceinline__ QuantParams qparams_for(int vmax, int bits, const QuantParams* __restrict__ tab) {
    if (tab && vmax >= 0 && vmax <= kQpTableMax && bits >= 2 && bits <= 8)
        return tab[(bits - 2) * (kQpTableMax + 1) + vmax];
    return derive_qparams_block(vmax, bits);
}

__device__ __forceinline__ QuantParams derive_qparams_warp(int vmax, int bits) {
    const int lane = threadIdx.x & 31;
    const int qmax = (1 << (bits - 1)) - 1;
    const double sa = fmax(double(vmax) / double(qmax), 1e-8);
    int e;
    frexp(sa, &e);
    const int S = 29 + e;  // mul lands in (2^29, 2^30]
    const long long m0 = (long long)floor(ldexp(1.0, S) / sa);
    int found = -1;
    for (int cand = 0; cand < 5 && found < 0; ++cand) {
        const long long mul = qcand(m0, cand);
        bool bad = mul <= 0;
        for (int k = lane; k <= qmax && !bad; k += 32) bad = qlevel_bad(k, vmax, sa, mul, S);
        if (!__any_sync(0xffffffffu, bad)) found = cand;
    }
    QuantParams p;
    p.sa = sa;
    p.shift = S;
    p.vmax = vmax;
    p.qmax = qmax;
    p.exact = found >= 0;
    p.mul = qcand(m0, found >= 0 ? found : 0);
    return p;
}

// clamp(rint(v), 0, 127) as int8: cvt.rni.s32.f64 (round-to-nearest-even like rint, saturating
// beyond int32, which the clamp maps to the same 0 / 127) and an integer clamp -- bit-identical
// to fmin(fmax(rint(v), 0.0), 127.0) for every non-NaN v, in three instructions.
__device__ __forceinline__ int8_t requant_i8(double v) {
    return int8_t(min(max(__double2int_rn(v), 0), 127));
}

// clamp(rint(y * sc * rq), 0, 127) with the conversions on the fp64 add pipe (the I2F / F2I
// conversion units are a quarter of its rate): double(y) = (2^52 + 2^31 + y) - (2^52 + 2^31)
// exactly, the products as in requant_i8(double(y) * sc * rq), and rint(t) as the low word of
// t + 1.5 * 2^52 (round to nearest even at unit ulp) -- valid while |t| < 2^31, which the caller
// guarantees with |sc * rq| < 1.
__device__ __forceinline__ int requant_i8_small(int y, double sc, double rq) {
    const double yd = __hiloint2double(0x43300000, y ^ int(0x80000000u)) - 4503601774854144.0;
    // (explicitly rounded products and sum: a fused t * rq + 1.5 * 2^52 would round the exact product,
    // not t, to an integer -- a different result when t lands exactly on a half-integer)
    const double t = __dmul_rn(__dmul_rn(yd, sc), rq);
    return __vimin_s32_relu(__double2loint(__dadd_rn(t, 6755399441055744.0)), 127);  // max(min(r, 127), 0)
}


}  // namespace sfcb200
