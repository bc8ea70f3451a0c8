// Microbenchmark: per-phase cost of a persistent grid synchronised by per-CTA
// epoch flags (no atomics), vs the atomic-counter grid barrier and the graph+PDL
// kernel chain (grid_sync_probe.cu). Each phase every thread reads two values a
// neighbour CTA wrote in the previous phase (double buffered) and writes its own.
//   mode 0: wait for the CTAs within +-span of this one
//   mode 1: wait for all CTAs (flag barrier: lanes poll disjoint flags)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_flags(int phases, int mode, int span, unsigned *flags, double *buf, int *err) {
    const int b = blockIdx.x, nb = gridDim.x, t = threadIdx.x, T = blockDim.x;
    const unsigned base = ld_acquire(&flags[b * 32]);  // epochs continue across launches
    for (int p = 1; p <= phases; ++p) {
        const unsigned want = base + p - 1;
        // wait for the producers of phase p-1
        if (mode == 0) {
            if (t < 2 * span + 1) {
                const int q = b - span + t;
                if (q >= 0 && q < nb && q != b) {
                    long spins = 0;
                    while (ld_acquire(&flags[q * 32]) < want)
                        if (++spins > (1l << 26)) { *err = 1; break; }
                }
            }
        } else {
            for (int q = t; q < nb; q += T) {
                if (q == b) continue;
                long spins = 0;
                while (ld_acquire(&flags[q * 32]) < want)
                    if (++spins > (1l << 26)) { *err = 1; break; }
            }
        }
        __syncthreads();
        const double *in = buf + ((p - 1) & 1) * (size_t)nb * T;
        double *out = buf + (p & 1) * (size_t)nb * T;
        const int l = (b > 0 ? b - 1 : nb - 1), r = (b + 1 < nb ? b + 1 : 0);
        const double v = (mode == 0 || true) ? in[l * T + t] + in[r * T + (T - 1 - t)] : 0.0;
        out[b * T + t] = 0.5 * v + 1.0;
        __syncthreads();
        if (t == 0) st_release(&flags[b * 32], want + 1);
    }
}

int main() {
    unsigned *flags; double *buf; int *err;
    cudaMalloc(&flags, 4096 * 128); cudaMemset(flags, 0, 4096 * 128);
    cudaMalloc(&buf, 64 << 20); cudaMemset(buf, 0, 64 << 20);
    cudaMalloc(&err, 4); cudaMemset(err, 0, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    struct Cfg { int grid, threads, mode, span; } cfgs[] = {
        {148, 256, 0, 1}, {148, 256, 0, 4}, {148, 256, 1, 0}, {296, 256, 0, 1}, {296, 256, 1, 0},
        {64, 256, 0, 1}, {64, 256, 1, 0}, {16, 256, 1, 0}, {148, 512, 0, 2}};
    for (auto c : cfgs) {
        cudaMemset(flags, 0, 4096 * 128);
        const int phases = 2000;
        k_flags<<<c.grid, c.threads>>>(10, c.mode, c.span, flags, buf, err);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k_flags<<<c.grid, c.threads>>>(phases, c.mode, c.span, flags, buf, err);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        int h = 0; cudaMemcpy(&h, err, 4, cudaMemcpyDeviceToHost);
        printf("grid %4d x %3d mode %d span %d: %.3f us per phase (err %d, %s)\n", c.grid, c.threads, c.mode, c.span,
               ms * 1e3 / phases, h, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
