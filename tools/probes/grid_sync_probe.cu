// Microbenchmark: cost of a software grid-wide barrier (one CTA per SM or 4 per
// SM, all resident) vs back-to-back dependent launches with PDL in a CUDA graph.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned g_count = 0;
__device__ volatile unsigned g_gen = 0;
__device__ __forceinline__ void grid_sync(unsigned nblocks, unsigned &gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned my = gen + 1;
        if (atomicAdd(&g_count, 1u) == nblocks - 1) {
            g_count = 0;
            __threadfence();
            g_gen = my;
        } else {
            while (g_gen < my) { }
        }
        __threadfence();
    }
    gen += 1;
    __syncthreads();
}
__global__ void k_sync(int iters, double *buf) {
    unsigned gen = g_gen;
    for (int i = 0; i < iters; ++i) {
        buf[blockIdx.x * blockDim.x + threadIdx.x] += 1.0;
        grid_sync(gridDim.x, gen);
    }
}
__global__ void k_step(double *buf) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    buf[blockIdx.x * blockDim.x + threadIdx.x] += 1.0;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
int main() {
    double *buf; cudaMalloc(&buf, 8 << 20); cudaMemset(buf, 0, 8 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int per : {1, 2, 4}) {
        const int grid = 148 * per, iters = 2000;
        k_sync<<<grid, 256>>>(10, buf); cudaDeviceSynchronize();
        cudaEventRecord(e0); k_sync<<<grid, 256>>>(iters, buf); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("grid barrier, %d CTAs: %.3f us (%s)\n", grid, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    cudaStream_t s; cudaStreamCreate(&s);
    for (int grid : {16, 148, 592}) {
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 200; ++i) {
            cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.stream = s;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_step, buf);
        }
        cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
        cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("graph+PDL chain, %d CTAs: %.3f us per kernel (%s)\n", grid, ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
