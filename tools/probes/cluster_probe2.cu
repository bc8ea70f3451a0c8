// Cluster phase cost with neighbour exchange through L2 (ld.global.cg) vs DSMEM
// (scattered and coalesced). nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned crank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
// MODE 0: L2 gathers (scattered over the whole vector); 1: DSMEM coalesced (lane-contiguous from one peer)
template <int K, int MODE>
__global__ void k(int iters, double *g, int n) {
    extern __shared__ double buf[];
    const unsigned me = crank();
    const int nt = blockDim.x * gridDim.x;
    const int gid = me * blockDim.x + threadIdx.x;
    buf[threadIdx.x] = gid;
    g[gid] = gid;
    csync();
    double acc = 0;
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < K; ++q) {
            if (MODE == 0) {
                const int j = (gid * 7 + q * 1031 + it) % nt;
                acc += __ldcg(g + j);
            } else {
                unsigned a = base + 8u * ((threadIdx.x + q) % blockDim.x), ra;
                unsigned peer = (me + 1 + q) % gridDim.x;
                asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(peer));
                double v;
                asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
                acc += v;
            }
        }
        if (MODE == 0) g[gid] = acc; else buf[threadIdx.x] = acc;
        csync();
    }
    if (acc == 12345.0) g[0] = acc;
}
template <int K, int M> void run(int ctas, int threads) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = 8 * threads;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ctas; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(k<K, M>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    double *g; cudaMalloc(&g, 8 * ctas * threads);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        int iters = 2000;
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k<K, M>, iters, g, ctas * threads);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("ctas %2d threads %4d loads %d %s: %.3f us per phase (%s)\n", ctas, threads, K,
                        M == 0 ? "L2-gather " : "DSMEM-coal", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(g);
}
int main() {
    for (int c : {16, 8}) for (int t : {256, 512, 1024}) { run<1, 0>(c, t); run<7, 0>(c, t); run<1, 1>(c, t); run<7, 1>(c, t); }
    return 0;
}
