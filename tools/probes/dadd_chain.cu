// Dependent fp64 add chain latency on sm_100a: plain DADD chain, and the
// shuffle-then-add pattern of warp_row_eval (8 shuffles ahead, 8 adds).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double *out, double y, int n, long long *cyc) {
    double s = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
        s = __dadd_rn(s, y);
        s = __dadd_rn(s, y);
        s = __dadd_rn(s, y);
        s = __dadd_rn(s, y);
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void shfl_chain(double *out, const double *p, int n, long long *cyc) {
    const int lane = threadIdx.x & 31;
    double v = p[lane];
    double s = 0.0;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j0 = 0; j0 < 32; j0 += 8) {
            double q[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = __shfl_sync(0xffffffffu, v, j0 + j);
#pragma unroll
            for (int j = 0; j < 8; ++j) s = __dadd_rn(s, q[j]);
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// products staged in shared memory, one lane sums them (LDS 8 ahead)
__global__ void smem_chain(double *out, const double *p, int n, long long *cyc) {
    __shared__ double sp[32];
    const int lane = threadIdx.x & 31;
    sp[lane] = p[lane];
    __syncwarp();
    double s = 0.0;
    long long t0 = clock64();
    if (lane == 0) {
#pragma unroll 1
        for (int i = 0; i < n; ++i) {
#pragma unroll
            for (int j0 = 0; j0 < 32; j0 += 8) {
                double q[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) q[j] = sp[j0 + j];
#pragma unroll
                for (int j = 0; j < 8; ++j) s = __dadd_rn(s, q[j]);
            }
        }
    }
    long long t1 = clock64();
    __syncwarp();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double *out, *p;
    long long *cyc, h;
    cudaMalloc(&out, 1024);
    cudaMalloc(&p, 1024);
    cudaMemset(p, 0, 1024);
    cudaMalloc(&cyc, 8);
    const int n = 1000;
    chain<<<1, 32>>>(out, 1.0, n, cyc);
    chain<<<1, 32>>>(out, 1.0, n, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent DADD: %.2f cycles/add\n", double(h) / (4.0 * n));
    shfl_chain<<<1, 32>>>(out, p, n, cyc);
    shfl_chain<<<1, 32>>>(out, p, n, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("shfl 8 ahead + DADD: %.2f cycles/element\n", double(h) / (32.0 * n));
    smem_chain<<<1, 32>>>(out, p, n, cyc);
    smem_chain<<<1, 32>>>(out, p, n, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS 8 ahead + DADD (one lane): %.2f cycles/element\n", double(h) / (32.0 * n));
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
