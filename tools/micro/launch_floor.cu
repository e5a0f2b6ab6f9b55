// Launch-floor microbenchmark: per-kernel cost of chains of (nearly) empty kernels in a
// CUDA graph -- plain stream order, PDL (programmatic stream serialization) and with a
// memset node in front -- for a few grid sizes.  Used to size the fixed per-launch cost
// the SFC conv pays per kernel on small layers.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p, int spin_ns) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (spin_ns) __nanosleep(spin_ns);
    if (threadIdx.x == 0 && blockIdx.x == 0 && p) p[0] += 1;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static float run(int grid, int block, bool pdl, bool memset, int chain, int spin) {
    int* d;
    cudaMalloc(&d, 64);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    const int reps = 50;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < reps; ++r) {
        if (memset) cudaMemsetAsync(d + 8, 0, 16, s);
        for (int i = 0; i < chain; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(block);
            cfg.stream = s;
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            a[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = a;
            cfg.numAttrs = (pdl && (i > 0 || !memset)) ? 1 : 0;
            cudaLaunchKernelEx(&cfg, k_empty, d, spin);
        }
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(e0, s);
    const int it = 20;
    for (int w = 0; w < it; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(d);
    cudaStreamDestroy(s);
    return ms * 1000.f / it / reps;  // us per chain
}

int main() {
    printf("per-chain us (chain of 4 kernels), columns: plain, pdl, memset+plain, memset+pdl\n");
    for (int grid : {1, 148, 320, 1184}) {
        printf("grid %5d:", grid);
        for (int mode = 0; mode < 4; ++mode) printf(" %7.2f", run(grid, 256, mode & 1, mode & 2, 4, 0));
        printf("\n");
    }
    printf("single kernel grid 320: plain %.2f  pdl %.2f\n", run(320, 256, false, false, 1, 0),
           run(320, 256, true, false, 1, 0));
    for (int spin : {500, 1000, 1500, 2000, 2500, 3000, 4000})
        printf("chain4 grid 320 spin %4d ns: plain %.2f pdl %.2f\n", spin, run(320, 256, false, false, 4, spin),
               run(320, 256, true, false, 4, spin));
    return 0;
}
