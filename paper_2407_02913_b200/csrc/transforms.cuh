// Scheduled 1-D SFC transforms (exact integer arithmetic).
//
//   fwd1d<V>:  y[k] = sum_s BT[k][s] x[s]      n inputs -> K transform channels
//   inv1d<V>:  y[t] = sum_k A[k][t]  p[k]      K channels -> M outputs
//
// The generic matrix form (one multiply-add per nonzero) is the definition; the
// specialisations below are addition schedules that exploit the symbolic-DFT
// structure and are exact rewrites of it:
//  * forward SFT-6 in 14 additions (the schedule of proj/src/poly.cpp:55-66,
//    sft6_apply_fast), the Karatsuba sum rows in 1 addition each
//    (row 3 = row 1 + row 2, row 6 = row 4 + row 5) and the correction rows as
//    single differences (catalog.cpp:183-190): 18 additions for 8 -> 10;
//  * inverse: with u1 = P2-P3, v1 = P1-P2, u2 = P6-P4, v2 = P5-P6 the six core
//    outputs are E/O + (+-)A_{t mod 3} + B_{t mod 3} where A, B are 2-term
//    combinations (period 3, sign flip every half period) -- ~24 operations for
//    10 -> 6 instead of ~54 multiply-adds.
// tests/test_transforms_host.py checks every schedule against the matrix form on
// the host; tests/test_gpu_parity.py checks the kernels bit-exactly end to end.
#pragma once
#include "sfc_tables.cuh"

namespace sfcb200 {

template <int V, class T>
__host__ __device__ __forceinline__ void fwd1d_generic(const T (&x)[Tab<V>::n], T (&y)[Tab<V>::K]) {
#pragma unroll
    for (int k = 0; k < Tab<V>::K; ++k) {
        T acc = 0;
#pragma unroll
        for (int s = 0; s < Tab<V>::n; ++s) acc += T(Tab<V>::bt(k, s)) * x[s];
        y[k] = acc;
    }
}

template <int V, class T>
__host__ __device__ __forceinline__ void inv1d_generic(const T (&p)[Tab<V>::K], T (&y)[Tab<V>::M]) {
#pragma unroll
    for (int t = 0; t < Tab<V>::M; ++t) {
        T acc = 0;
#pragma unroll
        for (int k = 0; k < Tab<V>::K; ++k)
            if (Tab<V>::a(k, t) != 0) acc += T(Tab<V>::a(k, t)) * p[k];
        y[t] = acc;
    }
}

// Core SFT-6 over window samples w0..w5 -> channels [X0, a1, b1, a1+b1, a2, b2, a2+b2, X3].
template <class T>
__host__ __device__ __forceinline__ void sft6_core(T w0, T w1, T w2, T w3, T w4, T w5, T* y) {
    const T a = w0 + w3, b = w1 + w4, c = w2 + w5;
    const T d = w0 - w3, e = w1 - w4, f = w2 - w5;
    y[0] = (a + b) + c;    // X0
    y[1] = d + e;          // a1
    y[2] = -(e + f);       // b1
    y[3] = y[1] + y[2];    // a1 + b1
    y[4] = a - c;          // a2
    y[5] = c - b;          // b2
    y[6] = y[4] + y[5];    // a2 + b2
    y[7] = (d - e) + f;    // X3
}

// Core inverse for N = 6 at cyclic positions 0..5 (channels 0..7 of A).
template <class T>
__host__ __device__ __forceinline__ void isft6_core(const T* p, T (&c)[6]) {
    const T u1 = p[2] - p[3], v1 = p[1] - p[2], u2 = p[6] - p[4], v2 = p[5] - p[6];
    const T A0 = 2 * u1 + v1, A1 = u1 - v1, A2 = -(u1 + 2 * v1);
    const T B0 = 2 * u2 + v2, B1 = -(u2 + 2 * v2), B2 = v2 - u2;
    const T E = p[0] + p[7], O = p[0] - p[7];
    c[0] = E + A0 + B0;
    c[1] = O + A1 + B1;
    c[2] = E + A2 + B2;
    c[3] = O - A0 + B0;
    c[4] = E - A1 + B1;
    c[5] = O - A2 + B2;
}

template <int V, class T>
__host__ __device__ __forceinline__ void fwd1d(const T (&x)[Tab<V>::n], T (&y)[Tab<V>::K]) {
    if constexpr (V == 1) {  // sfc6-6x6-3x3: n = 8, window x1..x6, corrections x0-x6, x7-x1
        sft6_core(x[1], x[2], x[3], x[4], x[5], x[6], y);
        y[8] = x[0] - x[6];
        y[9] = x[7] - x[1];
    } else if constexpr (V == 2) {  // sfc6-7x7-3x3: n = 9, rows 9 and 10 coincide
        sft6_core(x[1], x[2], x[3], x[4], x[5], x[6], y);
        y[8] = x[0] - x[6];
        y[9] = x[7] - x[1];
        y[10] = y[9];
        y[11] = x[8] - x[2];
    } else if constexpr (V == 0) {  // sfc4-4x4-3x3: n = 6, window x1..x4
        const T s0 = x[1] + x[3], s1 = x[2] + x[4];
        y[0] = s0 + s1;              // X0
        y[1] = s1 - s0;              // -X2
        y[2] = (x[1] - x[3]) + (x[4] - x[2]);   // a1 + b1
        y[3] = x[4] - x[2];          // b1
        y[4] = x[1] - x[3];          // a1
        y[5] = x[0] - x[4];
        y[6] = x[5] - x[1];
    } else {
        fwd1d_generic<V>(x, y);
    }
}

// Row sum of BT row k: the response of channel k to a constant input.
template <int V>
__host__ __device__ constexpr int bt_rowsum(int k) {
    int r = 0;
    for (int s = 0; s < Tab<V>::n; ++s) r += Tab<V>::bt(k, s);
    return r;
}

// fwd1d plus a constant per channel, y[k] = sum_s BT[k][s] x[s] + C[k], in the same number of
// additions as fwd1d where the constants fold into three-input adds (the register transform's
// horizontal pass: the +2^15 lane bias of the max/min and the input-bias correction).
template <int V, class T>
__host__ __device__ __forceinline__ void fwd1d_bias(const T (&x)[Tab<V>::n], T (&y)[Tab<V>::K], const T (&C)[Tab<V>::K]) {
    if constexpr (V == 1 || V == 2) {
        const T a = x[1] + x[4], b = x[2] + x[5], c = x[3] + x[6];
        const T d = x[1] - x[4], e = x[2] - x[5], f = x[3] - x[6];
        y[0] = (a + b) + (c + C[0]);
        y[1] = d + e + C[1];
        y[2] = C[2] - e - f;
        y[3] = y[1] + y[2] + (C[3] - C[1] - C[2]);
        y[4] = a - c + C[4];
        y[5] = c - b + C[5];
        y[6] = y[4] + y[5] + (C[6] - C[4] - C[5]);
        y[7] = (d + f + C[7]) - e;
        y[8] = x[0] - x[6] + C[8];
        y[9] = x[7] - x[1] + C[9];
        if constexpr (V == 2) {
            y[10] = x[7] - x[1] + C[10];
            y[11] = x[8] - x[2] + C[11];
        }
    } else if constexpr (V == 0) {
        const T s0 = x[1] + x[3], s1 = x[2] + x[4], a1 = x[1] - x[3], b1 = x[4] - x[2];
        y[0] = s0 + s1 + C[0];
        y[1] = s1 - s0 + C[1];
        y[2] = a1 + b1 + C[2];
        y[3] = b1 + C[3];
        y[4] = a1 + C[4];
        y[5] = x[0] - x[4] + C[5];
        y[6] = x[5] - x[1] + C[6];
    } else {
        fwd1d_generic<V>(x, y);
        for (int k = 0; k < Tab<V>::K; ++k) y[k] += C[k];
    }
}

template <int V, class T>
__host__ __device__ __forceinline__ void inv1d(const T (&p)[Tab<V>::K], T (&y)[Tab<V>::M]) {
    // Output t of the tile sits at cyclic position (t - offset) mod N with offset = 1,
    // i.e. c[(t + N - 1) % N] of the core inverse.
    if constexpr (V == 1) {  // M = 6; corrections: 6 P8 at t = 0, 6 P9 at t = 5
        T c[6];
        isft6_core(p, c);
        y[0] = c[5] + 6 * p[8];
        y[1] = c[0];
        y[2] = c[1];
        y[3] = c[2];
        y[4] = c[3];
        y[5] = c[4] + 6 * p[9];
    } else if constexpr (V == 2) {  // M = 7 (t = 6 is cyclic position 5 again); corrections rows 8..11
        T c[6];
        isft6_core(p, c);
        y[0] = c[5] + 6 * p[8];
        y[1] = c[0];
        y[2] = c[1];
        y[3] = c[2];
        y[4] = c[3];
        y[5] = c[4] + 6 * p[10];
        y[6] = c[5] + 6 * (p[9] + p[11]);
    } else if constexpr (V == 0) {  // M = 4: E/O = P0 +- P1, g = P2-P3-P4, h = P3-P4; 4 P5 at t=0, 4 P6 at t=3
        const T g = p[2] - p[3] - p[4], h = p[3] - p[4];
        const T e = p[0] + p[1], o = p[0] - p[1];
        y[0] = e + 2 * h + 4 * p[5];
        y[1] = o + 2 * g;
        y[2] = e - 2 * h;
        y[3] = o - 2 * g + 4 * p[6];
    } else {
        inv1d_generic<V>(p, y);
    }
}

}  // namespace sfcb200
