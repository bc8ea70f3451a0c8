// Launch-chain floor probe: per-kernel time of a CUDA graph of N dependent
// kernels (grid G x 256), with/without PDL, doing nothing / one dependent
// load->store per thread. nvcc -gencode arch=compute_100a,code=sm_100a -O3 chain_floor.cu -o chain_floor
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
struct Big {
    double v[140];
};
template <int WORK>
__global__ void kb(const double *__restrict__ a, double *__restrict__ b, const int *__restrict__ idx, int n,
                   const __grid_constant__ Big big) {
    extern __shared__ double sm[];
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int j = __ldg(idx + i);
    if (WORK >= 4) {
        if (threadIdx.x < 128) sm[threadIdx.x] = __ldg(a + threadIdx.x);
        __syncthreads();
    }
    pdl_wait();
    pdl_trigger();
    if (i < n) {
        double v = a[j] + big.v[threadIdx.x & 7] + (WORK >= 4 ? sm[threadIdx.x & 127] : 0.0);
        b[i] = WORK >= 5 ? __ddiv_rn(v, 3.0) : v * 1.0000001 + 1.0;
    }
}
template <int WORK>
__global__ void k(const double *__restrict__ a, double *__restrict__ b, const int *__restrict__ idx, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int j = 0;
    if (WORK >= 2 && i < n) j = __ldg(idx + i);  // constant: before the wait
    pdl_wait();
    pdl_trigger();
    if (WORK >= 1 && i < n) {
        double v = a[WORK >= 2 ? j : i];
        b[i] = v * 1.0000001 + 1.0;
    }
}
template <int WORK>
float run(int G, int N, bool pdl, double *a, double *b, int *idx) {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        double *x = (i & 1) ? b : a, *y = (i & 1) ? a : b;
        if constexpr (WORK >= 3) {
            Big big = {};
            cfg.dynamicSmemBytes = WORK >= 4 ? 1024 : 0;
            cudaLaunchKernelEx(&cfg, kb<WORK>, (const double *)x, y, (const int *)idx, G * 256, big);
        } else {
            cudaLaunchKernelEx(&cfg, k<WORK>, (const double *)x, y, (const int *)idx, G * 256);
        }
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    const int R = 10;
    for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(s);
    return ms * 1000.f / (R * N);
}
int main() {
    const int M = 1 << 22;
    double *a, *b;
    int *idx;
    cudaMalloc(&a, M * 8);
    cudaMalloc(&b, M * 8);
    cudaMalloc(&idx, M * 4);
    cudaMemset(a, 0, M * 8);
    cudaMemset(b, 0, M * 8);
    cudaMemset(idx, 0, M * 4);
    const int N = 200;
    for (int G : {16, 32, 64, 148, 296, 888}) {
        printf("G=%4d  empty: %.2f us (pdl %.2f)  ld/st: %.2f (pdl %.2f)  idx->ld/st: %.2f (pdl %.2f)  big %.2f  +smem %.2f  +div %.2f\n", G,
               run<0>(G, N, false, a, b, idx), run<0>(G, N, true, a, b, idx), run<1>(G, N, false, a, b, idx),
               run<1>(G, N, true, a, b, idx), run<2>(G, N, false, a, b, idx), run<2>(G, N, true, a, b, idx),
               run<3>(G, N, true, a, b, idx), run<4>(G, N, true, a, b, idx), run<5>(G, N, true, a, b, idx));
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
