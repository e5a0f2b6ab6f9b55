// Probe: how TMA lays a box with a 32-byte inner dimension into shared memory under
// CU_TENSOR_MAP_SWIZZLE_128B.  Source: bytes [F=16][T=4][96] (value = f*64 + t*16 + byte%16 ...
// encoded uniquely); box {32, 4, 16} at x = 32.  Hypothesis "address swizzle": the box is laid
// densely as [f][t][32 B] (128 B per f row) and 16-byte chunk c of row f lands at c ^ (f & 7).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2407_02913_b200/csrc tma_swz_probe.cu -o tma_swz_probe -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace sfcb200;

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, uint8_t* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    uint8_t* s = sm + ((1024u - (ptx::smem_u32(sm) & 1023u)) & 1023u);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbar_init();
        ptx::mbar_expect_tx(&bar, 32 * 4 * 16);
        ptx::tma_load_3d(s, &tm, &bar, 32, 0, 0);
        ptx::mbar_wait(&bar, 0);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) out[i] = s[i];
}

int main() {
    const int F = 16, T = 4, RB = 96;
    uint8_t h[F * T * RB];
    for (int f = 0; f < F; ++f)
        for (int t = 0; t < T; ++t)
            for (int b = 0; b < RB; ++b) h[(f * T + t) * RB + b] = uint8_t((f * 13 + t * 41 + b * 7) & 255);
    uint8_t *d, *o;
    cudaMalloc(&d, sizeof h);
    cudaMalloc(&o, 8192);
    cudaMemset(o, 0xee, 8192);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap tm;
    cuuint64_t dims[3] = {RB, T, F};
    cuuint64_t str[2] = {RB, RB * T};
    cuuint32_t box[3] = {32, 4, 16}, es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", int(r));
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    k_probe<<<1, 128, 8192>>>(tm, o);
    printf("launch %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    static uint8_t s[8192];
    cudaMemcpy(s, o, 8192, cudaMemcpyDeviceToHost);
    int bad_addr = 0, bad_dense = 0;
    for (int f = 0; f < F; ++f)
        for (int t = 0; t < T; ++t)
            for (int b = 0; b < 32; ++b) {
                const uint8_t want = h[(f * T + t) * RB + 32 + b];
                const int c = t * 2 + b / 16;
                if (s[f * 128 + ((c ^ (f & 7)) << 4) + (b & 15)] != want) ++bad_addr;
                if (s[f * 128 + t * 32 + b] != want) ++bad_dense;
            }
    printf("mismatches: address-swizzle hypothesis %d, unswizzled dense %d (of %d)\n", bad_addr, bad_dense, F * T * 32);
    for (int f = 0; f < 3; ++f)
        for (int t = 0; t < T; ++t)
            for (int c = 0; c < 2; ++c) {
                const uint8_t* want = h + (f * T + t) * RB + 32 + c * 16;
                int at = -1;
                for (int p = 0; p + 16 <= 8192; p += 16) {
                    bool eq = true;
                    for (int k = 0; k < 16; ++k) eq = eq && s[p + k] == want[k];
                    if (eq) { at = p; break; }
                }
                printf("f %d t %d chunk %d -> smem %d\n", f, t, c, at);
            }
    printf("first row bytes:");
    for (int i = 0; i < 32; ++i) printf(" %02x", s[i]);
    printf("\n");
    return 0;
}
