// Probe: 3-D TMA tile loads of an f64 grid (OOB fill): which encodings / coordinates work.
//   tma3d_probe bx by dtype(0 f64, 1 u64) x0 y0 z0 byversion(0/1)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k(const __grid_constant__ CUtensorMap m, int bx, int by, int cx, int cy, int cz, double *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    double *dst = reinterpret_cast<double *>(sm + 1024);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bx * by * 8));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                su32(dst)),
            "l"(reinterpret_cast<uint64_t>(&m)), "r"(cx), "r"(cy), "r"(cz), "r"(su32(bar))
            : "memory");
        asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(su32(bar)));
        out[0] = dst[bx + 1];
    }
}

int main(int argc, char **argv) {
    const int bx = atoi(argv[1]), by = atoi(argv[2]), dt = atoi(argv[3]), cx = atoi(argv[4]), cy = atoi(argv[5]),
              cz = atoi(argv[6]), byv = atoi(argv[7]);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t ge = byv ? cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q)
                         : cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const int nx = 20, ny = 20, nz = 20;
    double *g, *o;
    cudaMalloc(&g, 8 * nx * ny * nz);
    cudaMalloc(&o, 8);
    cudaMemset(g, 0, 8 * nx * ny * nz);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    CUtensorMap m;
    cuuint64_t dims[3] = {nx, ny, nz}, st[2] = {nx * 8, nx * ny * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, dt ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, st, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 32, 1024 + bx * by * 8>>>(m, bx, by, cx, cy, cz, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("box %dx%d dt %d at (%d,%d,%d) byver %d: getep %d q %d encode %d launch %s\n", bx, by, dt, cx, cy, cz, byv,
           (int)ge, (int)q, (int)r, cudaGetErrorString(e));
    return e != cudaSuccess;
}
