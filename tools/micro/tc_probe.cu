// Micro-probes that decide the fused-conv design (round 2):
//   1. tcgen05.ld (TMEM -> registers) throughput per SM for 4 / 8 / 16 warps;
//   2. tcgen05.mma kind::i8 (SS operands) throughput per SM vs N at M = 128;
//   3. legacy mma.sync m16n8k32 s8 throughput per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2407_02913_b200/csrc tc_probe.cu -o tc_probe -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace sfcb200;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void tmem_ld32_x(uint32_t taddr, int32_t (&r)[32]) { ptx::tmem_ld32(taddr, r); }

__global__ void k_ldtm(int iters, long long* cyc, int* sink, int shape) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc(&tbase, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t base = tbase;
    const int q = warp & 3;
    const int colblk = (warp >> 2) * 128 % 512;
    int acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        int32_t r[32];
        const uint32_t a = base + (uint32_t(q * 32) << 16) + uint32_t(colblk + (i & 3) * 32);
        ptx::tmem_ld32(a, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= r[j];
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 0x12345) sink[0] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(base, 512);
}

// Two loads in flight per wait.
__global__ void k_ldtm2(int iters, long long* cyc, int* sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc(&tbase, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t base = tbase;
    const int q = warp & 3;
    const int colblk = (warp >> 2) * 128 % 512;
    int acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 2) {
        int32_t r[32], s[32];
        const uint32_t a = base + (uint32_t(q * 32) << 16) + uint32_t(colblk);
        ptx::tmem_ld32(a, r);
        ptx::tmem_ld32(a + 32, s);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= r[j] + s[j];
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 0x12345) sink[0] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(base, 512);
}

__global__ void k_mma(int iters, int N, long long* cyc, int mode) {
    // mode 0: SS (A, B from shared memory); mode 1: A from TMEM (columns 256..), B from shared memory
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
    if (warp == 0) ptx::tmem_alloc(&tbase, 512);
    if (threadIdx.x == 32) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 32) {
        const uint32_t sa = ptx::smem_u32(smem), sb = ptx::smem_u32(smem + 32768);
        const uint32_t idesc = ptx::idesc_i8(128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int kk = i & 3;   // 4 K steps of 32 B within a 128B-swizzled row
            if (mode == 0) {
                ptx::mma_i8(tbase + uint32_t((i & 1) * 256), ptx::smem_desc_kmajor(sa + kk * 32, 128),
                            ptx::smem_desc_kmajor(sb + kk * 32, 128), idesc, 1);
            } else {
                const uint32_t ta = tbase + 256 + uint32_t(kk * 8);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tbase + uint32_t((i & 1) * 128)),
                    "r"(ta), "l"(ptx::smem_desc_kmajor(sb + kk * 32, 128)), "r"(idesc)
                    : "memory");
            }
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tbase, 512);
}

__global__ void k_mmasync(int iters, long long* cyc, int* sink) {
    int a[4] = {int(threadIdx.x), 1, 2, 3}, b[2] = {5, 7};
    int c[8][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    int s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    if (s == 0x1234567) sink[0] = s;
}

static double avg(long long* h, int n) { double s = 0; for (int i = 0; i < n; ++i) s += h[i]; return s / n; }

int main() {
    const int G = 148;
    long long *dc, hc[G];
    int* sink;
    CK(cudaMalloc(&dc, G * sizeof(long long)));
    CK(cudaMalloc(&sink, 4));
    const int iters = 4096;
    for (int w : {4, 8, 16}) {
        k_ldtm<<<G, 32 * w>>>(iters, dc, sink, 0);
        CK(cudaDeviceSynchronize());
        k_ldtm<<<G, 32 * w>>>(iters, dc, sink, 0);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost));
        double c = avg(hc, G);
        printf("ldtm 32x32b.x32 warps=%2d: %.1f cyc/iter  %.1f B/cyc/SM\n", w, c / iters, 4096.0 * w * iters / c);
        k_ldtm2<<<G, 32 * w>>>(iters, dc, sink);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost));
        c = avg(hc, G);
        printf("ldtm x32 x2-in-flight warps=%2d: %.1f B/cyc/SM\n", w, 4096.0 * w * iters / c);
    }
    CK(cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    for (int mode = 0; mode < 2; ++mode)
    for (int n : {8, 16, 24, 32, 48, 64, 128, 256}) {
        if (mode == 1 && n > 128) continue;
        const int it = 8192;
        k_mma<<<G, 128, 65536>>>(it, n, dc, mode);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        k_mma<<<G, 128, 65536>>>(it, n, dc, mode);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost));
        double c = avg(hc, G);
        printf("tcgen05.mma i8 %s M=128 N=%3d: %.2f cyc/mma  %.0f MAC/cyc/SM\n", mode ? "TS" : "SS", n, c / it, 128.0 * n * 32 * it / c);
    }
    for (int w : {4, 8, 16, 32}) {
        const int it = 2048;
        k_mmasync<<<G, 32 * w>>>(it, dc, sink);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost));
        double c = avg(hc, G);
        printf("mma.sync m16n8k32 s8 warps=%2d: %.0f MAC/cyc/SM\n", w, 16.0 * 8 * 32 * 8 * it * w / c);
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock %d kHz\n", clk);
    return 0;
}
