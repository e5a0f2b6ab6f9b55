// Batched fp64 contraction for the two paths tcgen05 cannot take (it has no fp64 kind):
//   P_f[t][o] = sum_c V_f[t][c] * U_f[o][c]        f < batch
// the exact-integer contraction of the 9-16 bit quantized path (|vq|, |uq| <= 2^15: every
// product and partial sum is an integer below 2^53, so the result is exact in any order and
// equals the reference's int64 pacc, quant.cpp:251-257) and the float fast_conv2d path
// (conv.cpp:466-509, compared at 1e-12).  Operands K-major as the rest of the pipeline lays
// them out: V [batch][Tpad][Cpad], U [batch][OCpad][Cpad], P [batch][Tpad][OCpad];
// Tpad % 128 == 0, OCpad % 64 == 0, Cpad % 64 == 0 (geom_init), so no bounds checks.
//
// CUDA-core DFMA kernel: 64 x 64 output tile per CTA, 256 threads with 4 x 4 outputs each,
// K staged 16 at a time in shared memory transposed to [k][row] (conflict-free reads of
// four consecutive rows per thread), double-buffered through registers.
#include <cuda_runtime.h>

#include "sfc_kernels.hpp"

namespace sfcb200 {
namespace {
constexpr int kTile = 64, kKs = 16, kThreads = 256;

__global__ void __launch_bounds__(kThreads) k_dgemm_nt(const double* __restrict__ U, const double* __restrict__ V,
                                                       double* __restrict__ P, int Tpad, int OCpad, int Cpad) {
    __shared__ double sV[2][kKs][kTile + 1];  // [k][t]
    __shared__ double sU[2][kKs][kTile + 1];  // [k][o]
    const int f = blockIdx.z, o0 = blockIdx.x * kTile, t0 = blockIdx.y * kTile;
    const double* Vf = V + size_t(f) * Tpad * Cpad + size_t(t0) * Cpad;
    const double* Uf = U + size_t(f) * OCpad * Cpad + size_t(o0) * Cpad;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;  // outputs (t0 + ty*4 + i, o0 + tx*4 + j)
    // loader: element e = tid + 256 * r (r = 0..3) of the 64 x 16 slab -> row e / 16, k e % 16
    double rv[4], ru[4];
    auto load = [&](int kc) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = tid + kThreads * r, row = e >> 4, k = e & 15;
            rv[r] = Vf[size_t(row) * Cpad + kc + k];
            ru[r] = Uf[size_t(row) * Cpad + kc + k];
        }
    };
    auto stash = [&](int b) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = tid + kThreads * r, row = e >> 4, k = e & 15;
            sV[b][k][row] = rv[r];
            sU[b][k][row] = ru[r];
        }
    };
    double acc[4][4] = {};
    load(0);
    stash(0);
    __syncthreads();
    int b = 0;
    for (int kc = 0; kc < Cpad; kc += kKs) {
        const bool more = kc + kKs < Cpad;
        if (more) load(kc + kKs);
#pragma unroll
        for (int k = 0; k < kKs; ++k) {
            double a[4], w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sV[b][k][ty * 4 + i], w[i] = sU[b][k][tx * 4 + i];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], w[j], acc[i][j]);
        }
        if (more) stash(b ^ 1);
        __syncthreads();
        b ^= 1;
    }
    double* Pf = P + size_t(f) * Tpad * OCpad;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) Pf[size_t(t0 + ty * 4 + i) * OCpad + o0 + tx * 4 + j] = acc[i][j];
}
}  // namespace

cudaError_t launch_dgemm_freq(const double* U, const double* V, double* P, int Tpad, int OCpad, int Cpad, int batch,
                              cudaStream_t st) {
    if (Tpad % kTile || OCpad % kTile || Cpad % kKs || batch <= 0) return cudaErrorInvalidValue;
    if (Tpad / kTile > 65535 || batch > 65535) return cudaErrorInvalidConfiguration;
    k_dgemm_nt<<<dim3(OCpad / kTile, Tpad / kTile, batch), kThreads, 0, st>>>(U, V, P, Tpad, OCpad, Cpad);
    return cudaGetLastError();
}

}  // namespace sfcb200
