// Microbenchmark: cost of a cluster-wide barrier phase (16 or 8 CTAs x T threads)
// with k DSMEM loads per thread per phase. nvcc -arch=sm_100a -O3 cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void csync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned crank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
template <int K, bool RELAXED>
__global__ void k(int iters, double *out) {
    extern __shared__ double buf[];
    const unsigned me = crank();
    const unsigned n = 16;  // cluster size bound
    buf[threadIdx.x] = threadIdx.x + me;
    csync();
    double acc = 0;
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < K; ++q) {
            unsigned a = base + 8u * ((threadIdx.x * 7 + q * 33) % blockDim.x), ra;
            unsigned peer = (me + 1 + q) % gridDim.x;
            asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(peer));
            double v;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
            acc += v;
        }
        buf[threadIdx.x] = acc;
        if (RELAXED) csync_relaxed(); else csync();
    }
    if (acc == 12345.0) out[0] = acc;
    (void)n;
}
template <int K, bool R> void run(int ctas, int threads) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = 8 * threads;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ctas; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(k<K, R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    double *out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        int iters = 2000;
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k<K, R>, iters, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("ctas %2d threads %4d loads/phase %d %s: %.3f us per phase (%s)\n", ctas, threads, K,
                        R ? "relaxed" : "release", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
int main() {
    for (int c : {16, 8, 4, 2}) for (int t : {256, 1024}) { run<0, false>(c, t); run<1, false>(c, t); run<7, false>(c, t); run<0, true>(c, t); }
    return 0;
}
