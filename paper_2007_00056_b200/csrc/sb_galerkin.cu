// GPU Galerkin coarse operator A_c = P^T A P for the unit piecewise-constant
// prolongation of a node-HEM aggregation (north star (c)).
//
// Reference: galerkin_product, inc/aggregation.hpp:92-152. Coarse row k
// accumulates, member by member in ascending fine order and entry by entry in
// CSR order, into one running sum per coarse column l = agg[col] that starts
// at 0.0; every touched column is stored (a 0.0 sum included) and the row's
// columns come out sorted. Here one thread owns one coarse row and performs
// exactly that sequence of additions (__dadd_rn, no reassociation), so A_c is
// bit-identical to the reference's (and to the host path, sb_host.cpp).
//
// Passes (all on the device): member pairs by atomic min/max (aggregates have
// 1 or 2 fine nodes under node-HEM), per-row distinct-column count, exclusive
// scan of the counts (row offsets), fill. Setup work, not the solve hot path:
// the kernels are simple and bounded by the fine matrix read (12 B/nnz + the
// agg[] gather per entry).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "sb_internal.h"

namespace sb {

#define GCK(x)                                                                                  \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw sb::cuda_error(std::string("galerkin: ") + #x + ": " + cudaGetErrorString(e_)); \
    } while (0)

constexpr int kGalCap = 64;  // expanded (column, value) pairs per coarse row held by one thread

__global__ void k_gal_members(int64_t n, const int32_t *__restrict__ agg, int64_t nc, int *__restrict__ cnt,
                              int *__restrict__ lo, int *__restrict__ hi, int *__restrict__ err) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = agg[i];
        if (c < 0 || c >= nc) {
            atomicExch(err, 1);
            continue;
        }
        atomicAdd(cnt + c, 1);
        atomicMin(lo + c, static_cast<int>(i));
        atomicMax(hi + c, static_cast<int>(i));
    }
}

// One coarse row: the reference's sparse accumulator, in registers / local memory.
// PASS 0 counts the distinct columns; PASS 1 writes the sorted row at rp_c[k].
template <int PASS>
__global__ void k_gal_rows(int64_t nc, const int *__restrict__ cnt, const int *__restrict__ lo,
                           const int *__restrict__ hi, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           const double *__restrict__ v, const int32_t *__restrict__ agg, int *__restrict__ rowcnt,
                           const int64_t *__restrict__ rp_c, int32_t *__restrict__ ci_c, double *__restrict__ v_c,
                           int *__restrict__ err) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nc;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int nm = cnt[k];
        if (nm < 1 || nm > 2) {
            atomicExch(err, 2);  // not a node-HEM aggregation (sizes 1..2)
            continue;
        }
        int cols[kGalCap];
        double acc[kGalCap];
        int nd = 0;
        bool over = false;
        for (int q = 0; q < nm && !over; ++q) {
            const int i = q == 0 ? lo[k] : hi[k];  // members in ascending fine order
            for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
                const int l = agg[ci[e]];
                int t = 0;
                while (t < nd && cols[t] != l) ++t;
                if (t == nd) {
                    if (nd == kGalCap) {
                        over = true;
                        break;
                    }
                    cols[nd] = l;
                    acc[nd] = 0.0;  // the reference's SPA slot starts at 0.0
                    ++nd;
                }
                if constexpr (PASS == 1) acc[t] = __dadd_rn(acc[t], v[e]);
            }
        }
        if (over) {
            atomicExch(err, 3);
            continue;
        }
        if constexpr (PASS == 0) {
            rowcnt[k] = nd;
        } else {
            // insertion sort of the touched columns (distinct keys: order is unique)
            for (int a = 1; a < nd; ++a) {
                const int c = cols[a];
                const double s = acc[a];
                int b = a - 1;
                while (b >= 0 && cols[b] > c) {
                    cols[b + 1] = cols[b];
                    acc[b + 1] = acc[b];
                    --b;
                }
                cols[b + 1] = c;
                acc[b + 1] = s;
            }
            const int64_t o = rp_c[k];
            for (int t = 0; t < nd; ++t) {
                ci_c[o + t] = cols[t];
                v_c[o + t] = acc[t];
            }
        }
    }
}

// Exclusive scan of int counts into int64 offsets (out[0] = 0, out[n] = total):
// per-block scans, a single-block scan of the block totals, then the add.
constexpr int kScanThreads = 1024, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *sh, int64_t *total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t s = lane < (blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sh[lane] = s;
    }
    __syncthreads();
    const int64_t before = (w > 0 ? sh[w - 1] : 0) + x - v;
    if (total) *total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

__global__ void k_scan_tiles(int64_t n, const int *__restrict__ in, int64_t *__restrict__ out, int64_t *__restrict__ tiles) {
    __shared__ int64_t sh[32];
    __shared__ int64_t tot;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
    int64_t loc[kScanItems], s = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
        loc[q] = (base + q < n) ? in[base + q] : 0;
        s += loc[q];
    }
    int64_t run = block_excl_scan(s, sh, threadIdx.x == 0 ? &tot : nullptr);
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
        if (base + q < n) out[base + q] = run;
        run += loc[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) tiles[blockIdx.x] = tot;
}

__global__ void k_scan_totals(int64_t ntiles, int64_t *__restrict__ tiles, int64_t *__restrict__ grand) {
    __shared__ int64_t sh[32];
    __shared__ int64_t tot;
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < ntiles; b0 += kScanThreads) {
        const int64_t i = b0 + threadIdx.x;
        const int64_t v = i < ntiles ? tiles[i] : 0;
        const int64_t e = block_excl_scan(v, sh, threadIdx.x == 0 ? &tot : nullptr);
        if (i < ntiles) tiles[i] = carry + e;
        __syncthreads();
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *grand = carry;
}

__global__ void k_scan_add(int64_t n, int64_t *__restrict__ out, const int64_t *__restrict__ tiles,
                           const int64_t *__restrict__ grand) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] += tiles[i / kScanTile];
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = *grand;
}

__global__ void k_fill_int(int64_t n, int *p, int v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

namespace {
struct DevBuf {
    void *p = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t bytes) { GCK(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    template <typename T> T *as() const { return static_cast<T *>(p); }
};
int grid_for(int64_t n, int threads) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16)));
}
} // namespace

// Host CSR in, host CSR out; every arithmetic step on the device.
HostCsr galerkin_gpu(const HostCsr &A, const std::vector<int32_t> &agg, int64_t nc, int device) {
    if (A.nnz() > INT32_MAX - 1 || A.n > INT32_MAX - 1)
        throw invalid_argument("galerkin_gpu: level too large for int32 device offsets");
    GCK(cudaSetDevice(device));
    const int64_t n = A.n, nnz = A.nnz();
    std::vector<int32_t> rp32(static_cast<size_t>(n) + 1);
    for (int64_t i = 0; i <= n; ++i) rp32[static_cast<size_t>(i)] = static_cast<int32_t>(A.rp[static_cast<size_t>(i)]);
    DevBuf d_rp(4 * (n + 1)), d_ci(4 * nnz), d_v(8 * nnz), d_agg(4 * n);
    DevBuf d_cnt(4 * nc), d_lo(4 * nc), d_hi(4 * nc), d_rowcnt(4 * nc), d_rpc(8 * (nc + 1)), d_err(4);
    const int64_t ntiles = (nc + kScanTile - 1) / kScanTile;
    DevBuf d_tiles(8 * std::max<int64_t>(ntiles, 1)), d_grand(8);
    GCK(cudaMemcpy(d_rp.p, rp32.data(), 4 * (n + 1), cudaMemcpyHostToDevice));
    GCK(cudaMemcpy(d_ci.p, A.ci.data(), 4 * nnz, cudaMemcpyHostToDevice));
    GCK(cudaMemcpy(d_v.p, A.v.data(), 8 * nnz, cudaMemcpyHostToDevice));
    GCK(cudaMemcpy(d_agg.p, agg.data(), 4 * n, cudaMemcpyHostToDevice));
    GCK(cudaMemset(d_cnt.p, 0, 4 * nc));
    GCK(cudaMemset(d_err.p, 0, 4));
    k_fill_int<<<grid_for(nc, 256), 256>>>(nc, d_lo.as<int>(), INT32_MAX);
    k_fill_int<<<grid_for(nc, 256), 256>>>(nc, d_hi.as<int>(), -1);
    k_gal_members<<<grid_for(n, 256), 256>>>(n, d_agg.as<int32_t>(), nc, d_cnt.as<int>(), d_lo.as<int>(),
                                             d_hi.as<int>(), d_err.as<int>());
    k_gal_rows<0><<<grid_for(nc, 128), 128>>>(nc, d_cnt.as<int>(), d_lo.as<int>(), d_hi.as<int>(), d_rp.as<int32_t>(),
                                              d_ci.as<int32_t>(), d_v.as<double>(), d_agg.as<int32_t>(),
                                              d_rowcnt.as<int>(), nullptr, nullptr, nullptr, d_err.as<int>());
    GCK(cudaGetLastError());
    int err = 0;
    GCK(cudaMemcpy(&err, d_err.p, 4, cudaMemcpyDeviceToHost));
    if (err == 1) throw invalid_argument("Aggregation: coarse index outside [0, n_coarse)");
    if (err == 2) throw invalid_argument("Aggregation: a coarse node has other than 1 or 2 fine nodes");
    if (err == 3) throw invalid_argument("galerkin_gpu: a coarse row touches more than 64 coarse columns");
    k_scan_tiles<<<static_cast<unsigned>(std::max<int64_t>(ntiles, 1)), kScanThreads>>>(
        nc, d_rowcnt.as<int>(), d_rpc.as<int64_t>(), d_tiles.as<int64_t>());
    k_scan_totals<<<1, kScanThreads>>>(ntiles, d_tiles.as<int64_t>(), d_grand.as<int64_t>());
    k_scan_add<<<grid_for(nc, 256), 256>>>(nc, d_rpc.as<int64_t>(), d_tiles.as<int64_t>(), d_grand.as<int64_t>());
    GCK(cudaGetLastError());
    int64_t nnz_c = 0;
    GCK(cudaMemcpy(&nnz_c, d_rpc.as<int64_t>() + nc, 8, cudaMemcpyDeviceToHost));
    DevBuf d_cic(4 * nnz_c), d_vc(8 * nnz_c);
    k_gal_rows<1><<<grid_for(nc, 128), 128>>>(nc, d_cnt.as<int>(), d_lo.as<int>(), d_hi.as<int>(), d_rp.as<int32_t>(),
                                              d_ci.as<int32_t>(), d_v.as<double>(), d_agg.as<int32_t>(), nullptr,
                                              d_rpc.as<int64_t>(), d_cic.as<int32_t>(), d_vc.as<double>(),
                                              d_err.as<int>());
    GCK(cudaGetLastError());
    HostCsr C;
    C.n = C.ncols = nc;
    C.rp.resize(static_cast<size_t>(nc) + 1);
    C.ci.resize(static_cast<size_t>(nnz_c));
    C.v.resize(static_cast<size_t>(nnz_c));
    GCK(cudaMemcpy(C.rp.data(), d_rpc.p, 8 * (nc + 1), cudaMemcpyDeviceToHost));
    GCK(cudaMemcpy(C.ci.data(), d_cic.p, 4 * nnz_c, cudaMemcpyDeviceToHost));
    GCK(cudaMemcpy(C.v.data(), d_vc.p, 8 * nnz_c, cudaMemcpyDeviceToHost));
    C.sync_rp32();
    return C;
}

} // namespace sb
