// B200-native solve phase: device hierarchy, sm_100a kernels, CUDA-graph
// Krylov drivers with device-side loop control, and the C ABI
// (include/sparsh_b200.h). See DESIGN.md for layout, kernels and rooflines.
//
// Reference (paths under /root/reference/proj/include/sparsh/):
//   spmv            csr.hpp:174-194      -> k_csr_tile<SPMV>
//   residual        csr.hpp:267-274      -> k_csr_tile<RESID>
//   Jacobi sweep    smoother.hpp:109-121 -> k_csr_tile<JACOBI>, k_jacobi_zero
//   restriction     cycle.hpp:69 (+ csr.hpp:226-241)  -> k_restrict
//   prolongation    cycle.hpp:72-73      -> k_prolong
//   coarse solve    coarse_solver.hpp:63-71,168-182  -> k_coarse_gemv
//   V-cycle         cycle.hpp:53-75      -> emit_vcycle
//   pcg             krylov.hpp:65-119    -> build_pcg_graph
//   pbicgstab       krylov.hpp:126-211   -> build_bicg_graph
//   amg_solve       cycle.hpp:91-130     -> build_amg_graph

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <cstdio>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <vector>
#include <unordered_map>
#include <thread>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "sb_internal.h"
#include "sb_kernels.cuh"

// Kernels that were built, measured slower than the defaults and kept for A/B
// work only: the plane-marching 27-point sweep (k_march),
// the pair-based residual + restriction (k_cross_rr) and the two-sweep
// temporal blocking (k_cross_tb2). They are templates instantiated only when
// the library is built with SB_EXPERIMENTAL=1 (make EXPERIMENTAL=1); the
// product build contains none of their code.
#ifndef SB_EXPERIMENTAL
#define SB_EXPERIMENTAL 0
#endif
constexpr bool kExperimental = SB_EXPERIMENTAL != 0;

namespace sb {

thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw sb::cuda_error(std::string(#x) + ": " + cudaGetErrorString(e_));              \
    } while (0)

// ===========================================================================
// device helpers
// ===========================================================================

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile("{\n"
                 ".reg .pred P1;\n"
                 "WAIT_%=:\n"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                 "@!P1 bra WAIT_%=;\n"
                 "}\n" ::"r"(smem_u32(bar)),
                 "r"(phase)
                 : "memory");
}
// Programmatic dependent launch: wait for the predecessor grid's completion
// (no-op when launched without the attribute) / allow the successor to launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifdef SB_XP_TRACE
// diagnostics build only (tools/xp_trace.py): per-CTA globaltimer stamps of
// k_crosspair (entry, after the dependency wait, exit)
__device__ unsigned long long g_xp_trace[6 * 65536];
__device__ unsigned g_xp_n;
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// grid-stride kernels: a CTA with at most one iteration over n items lets the
// dependent grid launch now (it still waits for this grid's completion); CTAs
// with more iterations trigger implicitly at exit
__device__ __forceinline__ void pdl_trigger_single(int64_t n) {
    if ((blockIdx.x + static_cast<int64_t>(gridDim.x)) * blockDim.x >= n) pdl_trigger();
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Deterministic block reduction of NV doubles (fixed shuffle tree, fixed warp
// order); the result is valid in thread 0.
template <int NV> __device__ __forceinline__ void block_reduce(double (&a)[NV], double *sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a[v] += __shfl_down_sync(0xffffffffu, a[v], off);
    if (lane == 0)
#pragma unroll
        for (int v = 0; v < NV; ++v) sh[v * 32 + warp] = a[v];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            a[v] = lane < nwarps ? sh[v * 32 + lane] : 0.0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) a[v] += __shfl_down_sync(0xffffffffu, a[v], off);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void record(DevState *st, int k, double v) {
    if (k < st->hist_cap) {
        st->hist_r[k] = v;
        st->hist_t[k] = static_cast<double>(globaltimer() - st->t0) * 1e-9;
    }
}

// Krylov scalar logic; runs in ONE thread after the grid-wide reduction.
// Each case restates the reference's scalar control flow (file:line noted).
__device__ void epilogue_logic(DevState *st, int op, double a, double b) {
    constexpr double eps = 1e-300;  // krylov.hpp:130
    constexpr double divf = 1e6;    // krylov.hpp:26
    switch (op) {
    case EP_PARTIAL:  // multi-rank: this rank's share, allreduced before the logic runs
        st->part[0] = a;
        st->part[1] = b;
        break;
    case EP_STORE:
        st->true_res = sqrt(a);
        break;
    case EP_INIT_NORM: {  // krylov.hpp:78-84 / 141-146, cycle.hpp:111-114
        const double rn = sqrt(a);
        st->rn = rn;
        st->r0 = rn;
        st->iter = 0;
        st->status = 0;
        st->half = 0;
        st->term = SB_MAX_ITERS;
        st->done = 0;
        st->true_res = rn;
        record(st, 0, rn);
        if (rn < st->tol) {
            st->term = SB_CONVERGED;
            st->done = 1;
        } else if (st->max_iters <= 0) {
            st->done = 1;
        }
        break;
    }
    case EP_PCG_RZ0:  // krylov.hpp:87
        st->rz = a;
        break;
    case EP_PCG_PAP:  // krylov.hpp:90-95
        if (st->done) break;
        st->pAp = a;
        if (a <= 0.0) {
            st->term = SB_BREAKDOWN;
            st->done = 1;
        } else {
            st->alpha = st->rz / a;
        }
        break;
    case EP_PCG_RN: {  // krylov.hpp:98-108
        if (st->done) break;
        const double rn = sqrt(a);
        const int it = st->iter + 1;
        st->rn = rn;
        record(st, it, rn);
        st->iter = it;
        if (rn < st->tol) {
            st->term = SB_CONVERGED;
            st->done = 1;
        } else if (rn > divf * st->r0) {
            st->term = SB_DIVERGED;
            st->done = 1;
        } else if (it >= st->max_iters) {
            st->done = 1;
        }
        break;
    }
    case EP_PCG_RZ:  // krylov.hpp:110-112
        if (st->done) break;
        st->beta = a / st->rz;
        st->rz = a;
        break;
    case EP_BI_RHO0:  // krylov.hpp:150-155
        st->rho = a;
        if (!st->done && fabs(a) < eps) {
            st->term = SB_BREAKDOWN;
            st->done = 1;
        }
        break;
    case EP_BI_DENOM:  // krylov.hpp:158-163
        if (st->done) break;
        st->denom = a;
        if (fabs(a) < eps) {
            st->term = SB_BREAKDOWN;
            st->done = 1;
        } else {
            st->alpha = st->rho / a;
        }
        break;
    case EP_BI_SN: {  // krylov.hpp:166-173
        if (st->done) break;
        const double sn = sqrt(a);
        st->sn = sn;
        if (sn < st->tol) {
            const int it = st->iter + 1;
            record(st, it, sn);
            st->iter = it;
            st->half = 1;
            st->term = SB_CONVERGED;
            st->done = 1;
        }
        break;
    }
    case EP_BI_AS:  // krylov.hpp:176-181
        if (st->done) break;
        if (a < eps) {
            st->term = SB_BREAKDOWN;
            st->done = 1;
        } else {
            st->omega = b / a;
        }
        break;
    case EP_BI_RN_RHO: {  // krylov.hpp:186-203 (+ the loop-top rho test, :152)
        if (st->done) break;
        const double rn = sqrt(a);
        const int it = st->iter + 1;
        st->rn = rn;
        record(st, it, rn);
        st->iter = it;
        if (rn < st->tol) {
            st->term = SB_CONVERGED;
            st->done = 1;
        } else if (rn > divf * st->r0) {
            st->term = SB_DIVERGED;
            st->done = 1;
        } else if (fabs(st->omega) < eps) {
            st->term = SB_BREAKDOWN;
            st->done = 1;
        } else {
            const double rho_next = b;
            st->beta = (rho_next / st->rho) * (st->alpha / st->omega);
            st->rho = rho_next;
            if (it >= st->max_iters) {
                st->done = 1;
            } else if (fabs(st->rho) < eps) {
                st->term = SB_BREAKDOWN;
                st->done = 1;
            }
        }
        break;
    }
    case EP_AMG_RN: {  // cycle.hpp:118-125
        if (st->done) break;
        const double rn = sqrt(a);
        const int it = st->iter + 1;
        st->rn = rn;
        st->true_res = rn;
        record(st, it, rn);
        st->iter = it;
        if (rn > divf * st->r0) {
            st->status = 2;
            st->done = 1;
        } else if (rn < st->tol) {
            st->term = SB_CONVERGED;
            st->done = 1;
        } else if (it >= st->max_iters) {
            st->done = 1;
        }
        break;
    }
    default:
        break;
    }
}

__device__ void epilogue(const Red &r, double a, double b) {
    epilogue_logic(r.st, r.op, a, b);
    for (int i = 0; i < r.cs.n; ++i)
        cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(r.cs.h[i]),
                                r.st->done ? 0u : 1u);
}

// Multi-rank: the scalar logic on the allreduced totals (st->red).
__global__ void k_logic(DevState *st, int op, CondSet cs) {
    pdl_wait();
    epilogue_logic(st, op, st->red[0], st->red[1]);
    for (int i = 0; i < cs.n; ++i)
        cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(cs.h[i]), st->done ? 0u : 1u);
}

// Grid-wide deterministic reduction + epilogue. Every thread of every block
// must call it (it contains barriers).
template <int NV> __device__ __forceinline__ void finish_reduction(const Red &r, double (&a)[NV]) {
    __shared__ double sh[2 * 32];
    __shared__ int am_last;
    block_reduce<NV>(a, sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) r.partials[2 * blockIdx.x + v] = a[v];
        __threadfence();
        const unsigned t = atomicAdd(r.counter, 1u);
        am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    double s[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) s[v] = 0.0;
    for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += blockDim.x)
#pragma unroll
        for (int v = 0; v < NV; ++v) s[v] += __ldcg(&r.partials[2 * b + v]);
    block_reduce<NV>(s, sh);
    if (threadIdx.x == 0) {
        *r.counter = 0u;
        epilogue(r, s[0], NV > 1 ? s[NV > 1 ? 1 : 0] : 0.0);
    }
}

// ===========================================================================
// CSR tile kernel: SpMV / residual / Jacobi sweep (+ optional fused dot)
// ===========================================================================

enum CsrMode {
    M_SPMV = 0,          // y = A x                          (csr.hpp:174-194)
    M_RESID = 1,         // r = f - A x                      (csr.hpp:267-274)
    M_JACOBI = 2,        // x' = x + w (f - A x) / a_ii      (smoother.hpp:113-120)
    // 3: retired (the first sweep from x = 0 is written by the parent's restriction)
    M_JACOBI_PROLONG = 4, // prolongation + first post-sweep fused: x_j + (0 + x_c[agg_j])
    M_RESID_RESTRICT = 5  // k_crosspair on a level whose aggregates are its row pairs: the pair's
                          // residuals -> f_c = (0 + r_2c) + r_2c+1 and the coarse first sweep
};

// Operands of the fused modes.
struct Aux {
    const double *diag;   // a_ii
    const int32_t *agg;   // fine_to_coarse (M_JACOBI_PROLONG)
    const double *xc;     // coarse correction (M_JACOBI_PROLONG)
};

// Mutable vectors inside the cluster tail kernel are read with ld.global.cg
// (L2; another CTA of the cluster may have rewritten them since the last
// phase); everywhere else with the read-only path.
template <bool CG> __device__ __forceinline__ double ldv(const double *p) {
    if constexpr (CG) return __ldcg(p);
    else return __ldg(p);
}

// The value the reference's sweep sees for x_j (bitwise).
template <int MODE, bool CG>
__device__ __forceinline__ double xval(int j, const double *x, const double *f, const Aux &a, double omega) {
    if constexpr (MODE == M_JACOBI_PROLONG)
        return __dadd_rn(ldv<CG>(x + j), __dadd_rn(0.0, ldv<CG>(a.xc + __ldg(a.agg + j))));
    else
        return ldv<CG>(x + j);
}

// Matrix entry storage formats (per level, chosen at upload):
//   VF 0: f64 values; 1: uint8 index into a <=256-entry dictionary of the
//         level's distinct values (exact doubles: lossless)
//   CF 0: int32 columns; 1: int16 column - row deltas (when every |delta| fits)
template <int VF, int CF> struct Ent {
    const void *vals;
    const void *cols;
    const double *dict;
    __device__ __forceinline__ int col(int k, int row) const {
        if constexpr (CF == 1) return row + static_cast<int>(static_cast<const int16_t *>(cols)[k]);
        else return static_cast<const int32_t *>(cols)[k];
    }
    __device__ __forceinline__ double val(int k) const {
        if constexpr (VF == 1) return dict[static_cast<const uint8_t *>(vals)[k]];
        else return static_cast<const double *>(vals)[k];
    }
};

// One row in the reference's order: sum = 0.0; sum += a_k * x_{c_k} for k in
// CSR order (no FMA), then the mode's epilogue.
template <int MODE, bool CG, int U = 8, typename E>
__device__ __forceinline__ double row_eval(int row, int rs, int re, const E &e, const double *x,
                                           const double *f, double fi, const Aux &aux, double omega) {
    double sum = 0.0, d = 0.0;
    double xi = 0.0;  // own iterate, loaded up front so its latency overlaps the row
    if constexpr (MODE >= M_JACOBI) xi = xval<MODE, CG>(row, x, f, aux, omega);
    for (int k = rs; k < re; k += U) {
        int c[U];
        double a[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k + u < re) {
                c[u] = e.col(k + u, row);
                a[u] = e.val(k + u);
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k + u < re) xv[u] = xval<MODE, CG>(c[u], x, f, aux, omega);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k + u < re) {
                sum = __dadd_rn(sum, __dmul_rn(a[u], xv[u]));
                if (MODE >= M_JACOBI && c[u] == row) d = a[u];
            }
    }
    if constexpr (MODE == M_SPMV) return sum;
    else if constexpr (MODE == M_RESID) return __dsub_rn(fi, sum);
    else return __dadd_rn(xi, __ddiv_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), d));
}

// Rows longer than this are evaluated by a whole warp (k_csr_tile).
constexpr int kLongRow = 32;
#ifndef SB_TILE_U
#define SB_TILE_U 4  // gathers in flight per row step in k_csr_tile (G128: 4 -> 67.0 ms, 6 -> 67.5, 8 -> 70.3 with spills, 2 -> 70.9, 16 -> 93.3)
#endif
// Rows longer than this (up to kHubMax per CTA; e.g. the hub row a stalled
// coarsening leaves: ~560 entries on G128's deep levels) are deferred to the
// end of k_csr_tile and evaluated by the whole CTA: every product at once into
// shared memory, then one thread per row adds them in CSR order (~8 cycles per
// entry). With a warp they paid a gather round trip per 32 entries: ~10 us
// per sweep on those levels.
#ifndef SB_HUB_ROW
#define SB_HUB_ROW 32  // measured on G128: 32 (every warp-path row) 70.3 ms, 96: 71.5, 256: 74.0, warp path only: 83.9
#endif
constexpr int kHubRow = SB_HUB_ROW;
constexpr int kHubMax = 16;  // deferred hub rows per CTA (more: the warp path)

// row_eval of one long row by a warp: lane l multiplies entries k0 + l (the
// products are the reference's, __dmul_rn), then every lane adds the 32
// products in CSR order from the shuffles (the same dependent chain of
// __dadd_rn as row_eval; the gathers of 32 entries are in flight together).
template <int MODE, typename E>
__device__ __forceinline__ double warp_row_eval(int row, int rs, int re, const E &e, const double *x,
                                                const double *f, double fi, const Aux &aux, double omega, int lane) {
    double sum = 0.0, d = 0.0;
#pragma unroll 1
    for (int k0 = rs; k0 < re; k0 += 32) {
        const int k = k0 + lane;
        double p = 0.0;
        bool isd = false;
        double a = 0.0;
        if (k < re) {
            const int c = e.col(k, row);
            a = e.val(k);
            p = __dmul_rn(a, xval<MODE, false>(c, x, f, aux, omega));
            isd = c == row;
        }
        const int cnt = min(32, re - k0);
        if (cnt == 32) {  // full chunk: shuffles issue 8 ahead of the dependent adds
#pragma unroll
            for (int j0 = 0; j0 < 32; j0 += 8) {
                double q[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) q[j] = __shfl_sync(0xffffffffu, p, j0 + j);
#pragma unroll
                for (int j = 0; j < 8; ++j) sum = __dadd_rn(sum, q[j]);
            }
        } else {
#pragma unroll 1
            for (int j = 0; j < cnt; ++j) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, p, j));
        }
        const unsigned dm = __ballot_sync(0xffffffffu, isd);
        if (MODE >= M_JACOBI && dm) d = __shfl_sync(0xffffffffu, a, 31 - __clz(dm));
    }
    if constexpr (MODE == M_SPMV) return sum;
    else if constexpr (MODE == M_RESID) return __dsub_rn(fi, sum);
    else {
        const double xi = xval<MODE, false>(row, x, f, aux, omega);
        return __dadd_rn(xi, __ddiv_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), d));
    }
}

// Persistent, double-buffered CSR tile pipeline. Tiles of <= 256 consecutive
// rows (tile_ptr, built at setup) are dealt round-robin to a grid sized to the
// SM count; for each tile one elected thread issues two TMA bulk copies
// (values + column indices, 16-byte aligned windows of the tile's contiguous
// nnz range) into the NEXT stage while the CTA computes the current one, so
// HBM streaming overlaps the x-gathers and arithmetic. Thread t owns row
// r0 + t and walks it in CSR order from shared memory. A tile whose nnz exceed
// the stage capacity (a single very long row) reads straight from global.
constexpr int kStages = 3;      // TMA pipeline depth (tiles in flight per CTA)
constexpr int kRpWin = 264;     // staged row-pointer window (ints): 256 + 1 + alignment
constexpr int kFWin = 258;      // staged f window (doubles): 256 + alignment

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Stage layout: [values][cols][rp kRpWin i32][f kFWin f64], each a 16-byte
// aligned window; sizes depend on the level's storage format.
__host__ __device__ __forceinline__ size_t stage_vbytes(int cap, int vf) {
    return vf ? static_cast<size_t>((cap + 31) & ~15) : static_cast<size_t>((cap + 3) & ~1) * 8;
}
__host__ __device__ __forceinline__ size_t stage_cbytes(int cap, int cf) {
    return cf ? static_cast<size_t>((cap + 15) & ~7) * 2 : static_cast<size_t>((cap + 11) & ~3) * 4;
}
__host__ __device__ __forceinline__ size_t stage_bytes_of(int cap, int vf, int cf) {
    return stage_vbytes(cap, vf) + stage_cbytes(cap, cf) + static_cast<size_t>(kRpWin) * 4 +
           static_cast<size_t>(kFWin) * 8;
}

#ifndef SB_TILE_MINB
#define SB_TILE_MINB 3
#endif
template <int MODE, int NV, int VF, int CF>
__global__ void __launch_bounds__(kTileRows, SB_TILE_MINB)
    k_csr_tile(const int32_t *__restrict__ rp, const void *__restrict__ cols, const void *__restrict__ vals,
               const double *__restrict__ dict, int ndict, const int32_t *__restrict__ tile_ptr, int ntiles,
               const double *__restrict__ x, const double *__restrict__ f, double *__restrict__ out,
               double omega, int cap, const int *skip, Aux aux, Red red) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[kStages];
    __shared__ __align__(8) uint64_t empty[kStages];
    __shared__ int4 hdr[kStages];
    __shared__ double sdict[VF ? 256 : 1];
    __shared__ int hub_rows[kHubMax];
    __shared__ int hub_off[kHubMax + 1];
    __shared__ int nhub;
    __shared__ double hub_d[kHubMax];
    double acc[NV > 0 ? NV : 1];
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) acc[v] = 0.0;

    auto emit_row = [&](int row, double o) {
        out[row] = o;
        if (NV >= 1) acc[0] += o * (red.w0 ? red.w0[row] : o);
        if (NV >= 2) acc[NV >= 2 ? 1 : 0] += o * (red.w1 ? red.w1[row] : o);
    };
    constexpr int VB = VF ? 1 : 8;  // bytes per value / column entry
    constexpr int CB = CF ? 2 : 4;
    constexpr int VA = 16 / VB, CA = 16 / CB;  // entries per 16-byte granule
    const size_t sb = stage_bytes_of(cap, VF, CF);
    const size_t o_c = stage_vbytes(cap, VF);
    const size_t o_rp = o_c + stage_cbytes(cap, CF);
    const size_t o_f = o_rp + static_cast<size_t>(kRpWin) * 4;
    constexpr int kWarps = kTileRows / 32;
    const unsigned char *vbase = static_cast<const unsigned char *>(vals);
    const unsigned char *cbase = static_cast<const unsigned char *>(cols);

    // thread 0: stage tile t into buffer s. Matrix data (values, columns, row
    // pointers) is constant and may be issued before the dependency wait;
    // with_f adds the rhs window (a predecessor output) once that wait is done.
    auto issue = [&](int t, int s, bool with_f) {
        const int r0 = tile_ptr[t], r1 = tile_ptr[t + 1];
        const int e0 = rp[r0], e1 = rp[r1];
        hdr[s] = make_int4(r0, r1, e0, e1);
        unsigned char *st = smem + s * sb;
        const bool staged = e1 - e0 <= cap && e1 > e0;
        const int va0 = e0 & ~(VA - 1), ca0 = e0 & ~(CA - 1), ra0 = r0 & ~3, fa0 = r0 & ~1;
        const uint32_t vbytes = staged ? static_cast<uint32_t>(((e1 + VA - 1) & ~(VA - 1)) - va0) * VB : 0u;
        const uint32_t cbytes = staged ? static_cast<uint32_t>(((e1 + CA - 1) & ~(CA - 1)) - ca0) * CB : 0u;
        const uint32_t rbytes = static_cast<uint32_t>(((r1 + 1 + 3) & ~3) - ra0) * 4u;
        const uint32_t fbytes = (MODE != M_SPMV && with_f) ? static_cast<uint32_t>((r1 & ~1) - fa0) * 8u : 0u;
        mbar_expect_tx(&full[s], vbytes + cbytes + rbytes + fbytes);
        if (vbytes) bulk_g2s(st, vbase + static_cast<size_t>(va0) * VB, vbytes, &full[s]);
        if (cbytes) bulk_g2s(st + o_c, cbase + static_cast<size_t>(ca0) * CB, cbytes, &full[s]);
        bulk_g2s(st + o_rp, rp + ra0, rbytes, &full[s]);
        if (fbytes) bulk_g2s(st + o_f, f + fa0, fbytes, &full[s]);
    };

    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < kStages; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kWarps);
        }
        fence_mbar_init();
    }
    if constexpr (VF == 1)
        for (int i = threadIdx.x; i < ndict; i += blockDim.x) sdict[i] = dict[i];
    if (threadIdx.x == 0) nhub = 0;
    __syncthreads();
    const int G = static_cast<int>(gridDim.x);
    const int b = static_cast<int>(blockIdx.x);
    // prologue tiles go out before the dependency wait WITHOUT f; their f rows
    // are read from global after the wait
    if (threadIdx.x == 0)
        for (int q = 0; q < kStages - 1; ++q)
            if (b + q * G < ntiles) issue(b + q * G, q, false);
    pdl_wait();  // predecessor complete: x, f (and skip) are final
    const bool active = !(skip && *skip);
    if (!active) {  // skipped (solve already finished): drain the prologue's copies
        for (int q = 0; q < kStages - 1; ++q)
            if (b + q * G < ntiles) mbar_wait(&full[q], 0u);
        pdl_trigger();
    } else {
        uint32_t fph = 0u, eph = 0u;  // parities of full[] (all threads) / empty[] (thread 0)
        int s = 0, it = 0;
        const int lane = threadIdx.x & 31;
        for (int t = b; t < ntiles; t += G, ++it, s = (s + 1 == kStages) ? 0 : s + 1) {
            if (t + G >= ntiles) pdl_trigger();  // last tile of this CTA: let the next kernel launch
            const int tn = t + (kStages - 1) * G;
            const int sn = (s + kStages - 1) % kStages;
            if (threadIdx.x == 0 && tn < ntiles) {
                if (it >= 1) {  // stage sn was consumed in iteration it-1
                    mbar_wait(&empty[sn], (eph >> sn) & 1u);
                    eph ^= 1u << sn;
                }
                issue(tn, sn, true);
            }
            mbar_wait(&full[s], (fph >> s) & 1u);
            fph ^= 1u << s;
            const int4 h = hdr[s];
            const int r0 = h.x, r1 = h.y;
            const int row = r0 + static_cast<int>(threadIdx.x);
            const unsigned char *st = smem + s * sb;
            const bool staged = (h.w - h.z) <= cap;
            Ent<VF, CF> e;
            e.vals = staged ? static_cast<const void *>(st - static_cast<size_t>(h.z & ~(VA - 1)) * VB) : vals;
            e.cols = staged ? static_cast<const void *>(st + o_c - static_cast<size_t>(h.z & ~(CA - 1)) * CB) : cols;
            e.dict = sdict;
            const int32_t *srp = reinterpret_cast<const int32_t *>(st + o_rp) - (r0 & ~3);
            auto rhs_of = [&](int rr) {  // f_row: staged window or global
                if (MODE == M_SPMV) return 0.0;
                const bool f_staged = it >= kStages - 1 && rr < (r1 & ~1);
                return f_staged ? reinterpret_cast<const double *>(st + o_f)[rr - (r0 & ~1)] : f[rr];
            };
            // rows longer than kLongRow go to the whole warp (below)
            const unsigned lm = __ballot_sync(0xffffffffu, row < r1 && srp[row + 1] - srp[row] > kLongRow);
            if (row < r1 && !((lm >> lane) & 1u))
                emit_row(row, row_eval<MODE, false, SB_TILE_U>(row, srp[row], srp[row + 1], e, x, f, rhs_of(row), aux, omega));
            for (unsigned m = lm; m; m &= m - 1) {  // gathers 32 entries at a time, sum in CSR order
                const int src = __ffs(m) - 1;
                const int lr = row - lane + src;
                if (srp[lr + 1] - srp[lr] > kHubRow) {  // deferred to the CTA (below), if there is room
                    int slot = 0;
                    if (lane == 0) slot = atomicAdd(&nhub, 1);
                    slot = __shfl_sync(0xffffffffu, slot, 0);
                    if (slot < kHubMax) {
                        if (lane == 0) hub_rows[slot] = lr;
                        continue;
                    }
                }
                const double o = warp_row_eval<MODE>(lr, srp[lr], srp[lr + 1], e, x, f, rhs_of(lr), aux, omega, lane);
                if (lane == src) emit_row(lr, o);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
        }
        // deferred hub rows: the whole CTA forms the products (every gather in
        // flight at once) into the drained stage buffers, then thread q adds row
        // q's products in CSR order. Every issued stage was consumed above, so
        // no copy is in flight.
        __syncthreads();
        const int nh = min(nhub, kHubMax);
        if (nh > 0) {
            double *buf = reinterpret_cast<double *>(smem);
            const int seg = static_cast<int>(kStages * sb / 8 < 8192 ? kStages * sb / 8 : 8192);
            Ent<VF, CF> eg;
            eg.vals = vals;
            eg.cols = cols;
            eg.dict = sdict;
            if (threadIdx.x == 0) {
                int o = 0;
                for (int q = 0; q < nh; ++q) {
                    hub_off[q] = o;
                    o += rp[hub_rows[q] + 1] - rp[hub_rows[q]];
                    hub_d[q] = 0.0;
                }
                hub_off[nh] = o;
            }
            __syncthreads();
            auto finish = [&](int q, double sum) {
                const int hr = hub_rows[q];
                const double fi = (MODE == M_SPMV) ? 0.0 : f[hr];
                double o;
                if constexpr (MODE == M_SPMV) o = sum;
                else if constexpr (MODE == M_RESID) o = __dsub_rn(fi, sum);
                else
                    o = __dadd_rn(xval<MODE, false>(hr, x, f, aux, omega),
                                  __ddiv_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), hub_d[q]));
                emit_row(hr, o);
            };
            auto add_chain = [&](const double *b, int len, double sum) {
                int k = 0;
                for (; k + 8 <= len; k += 8) {
                    double t[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) t[j] = b[k + j];
#pragma unroll
                    for (int j = 0; j < 8; ++j) sum = __dadd_rn(sum, t[j]);
                }
                for (; k < len; ++k) sum = __dadd_rn(sum, b[k]);
                return sum;
            };
            if (hub_off[nh] <= seg) {  // all rows at once: products, then one thread per row adds
                for (int k = threadIdx.x; k < hub_off[nh]; k += blockDim.x) {
                    int q = 0;
                    while (hub_off[q + 1] <= k) ++q;
                    const int hr = hub_rows[q];
                    const int ke = rp[hr] + (k - hub_off[q]);
                    const int c = eg.col(ke, hr);
                    const double a = eg.val(ke);
                    buf[k] = __dmul_rn(a, xval<MODE, false>(c, x, f, aux, omega));
                    if (MODE >= M_JACOBI && c == hr) hub_d[q] = a;
                }
                __syncthreads();
                if (static_cast<int>(threadIdx.x) < nh) {
                    const int q = threadIdx.x;
                    finish(q, add_chain(buf + hub_off[q], hub_off[q + 1] - hub_off[q], 0.0));
                }
            } else {  // row by row in segments of the buffer
                for (int q = 0; q < nh; ++q) {
                    const int hr = hub_rows[q];
                    const int rs = rp[hr], re = rp[hr + 1];
                    double sum = 0.0;
                    for (int s0 = rs; s0 < re; s0 += seg) {
                        const int s1 = min(re, s0 + seg);
                        __syncthreads();  // the previous segment's adds are done with buf
                        for (int k = s0 + static_cast<int>(threadIdx.x); k < s1; k += blockDim.x) {
                            const int c = eg.col(k, hr);
                            const double a = eg.val(k);
                            buf[k - s0] = __dmul_rn(a, xval<MODE, false>(c, x, f, aux, omega));
                            if (MODE >= M_JACOBI && c == hr) hub_d[q] = a;
                        }
                        __syncthreads();
                        if (threadIdx.x == 0) sum = add_chain(buf, s1 - s0, sum);
                    }
                    if (threadIdx.x == 0) finish(q, sum);
                }
            }
        }
    }
    if constexpr (NV > 0) finish_reduction<NV>(red, acc);
}

// ===========================================================================
// Grouped sliced-ELL ("SELL-G") pipeline: the default streamed format of every
// level whose slices pad by <= 50%. A slice holds H = 256 consecutive
// rows; its block in HBM is contiguous and 16-byte aligned:
//   hdr  int32 {ng, nfull, 0, 0}: groups, and groups every row fills (no masking)
//   vals [ng][H][GS]  (uint8 dictionary indices, or f64 values)
//   cols [ng][H][GS]  (int16 column - row deltas, or int32 columns)
//   meta [H] uint16   row length | (dictionary index of a_ii, or its slot) << 8
// so thread t reads GS consecutive entries of its row with ONE vector LDS per
// array (conflict-free) and the whole block arrives with ONE TMA bulk copy.
// Entries of a row keep the CSR order; slots >= the row length are predicated
// out of the sum, which therefore sees exactly the reference's operands in
// the reference's order (inc/csr.hpp:185-191): results are bitwise the
// reference's. The Jacobi division uses the Markstein correction with the
// host-rounded reciprocal of the (dictionary) diagonal, which is the
// correctly rounded quotient (IEEE a / a_ii) wherever no intermediate can
// under/overflow; other operands take __ddiv_rn.
// ===========================================================================

#ifndef SB_SG_STAGES
#define SB_SG_STAGES 4
#endif
constexpr int kSgStages = SB_SG_STAGES;  // slices in flight per CTA (power of two)

__host__ __device__ __forceinline__ int sg_entry_bytes(int vf, int cf) { return (vf ? 1 : 8) + (cf ? 2 : 4); }
constexpr int kSgHdr = 16;  // slice header: int32 {groups, unmasked groups, 0, 0}
__host__ __device__ __forceinline__ size_t sg_block_bytes(int ng, int gs, int h, int vf, int cf) {
    return kSgHdr + static_cast<size_t>(ng) * h * gs * sg_entry_bytes(vf, cf) + 2 * static_cast<size_t>(h);
}
__host__ __device__ __forceinline__ size_t sg_stage_bytes(int ngmax, int gs, int h, int vf, int cf) {
    return (sg_block_bytes(ngmax, gs, h, vf, cf) + 15) / 16 * 16 + 8 * static_cast<size_t>(h) /* f */;
}

template <int N> struct RawVec;
template <> struct RawVec<2> { using T = uint16_t; };
template <> struct RawVec<4> { using T = uint32_t; };
template <> struct RawVec<8> { using T = uint2; };
template <> struct RawVec<16> { using T = uint4; };
template <> struct RawVec<32> { struct alignas(16) T { uint4 a, b; }; };

template <int N> __device__ __forceinline__ uint32_t word_of(const typename RawVec<N>::T &v, int i) {
    if constexpr (N == 2) return v;
    else if constexpr (N == 4) return v;
    else if constexpr (N == 8) return i == 0 ? v.x : v.y;
    else if constexpr (N == 16) return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
    else {
        const uint4 &q = i < 4 ? v.a : v.b;
        const int j = i & 3;
        return j == 0 ? q.x : j == 1 ? q.y : j == 2 ? q.z : q.w;
    }
}

// a / d correctly rounded; y = RN(1/d) computed on the host (0 = unknown).
// q = RN(a y); r = a - d q (exact by FMA); q' = RN(q + r y) = RN(a / d)
// (Markstein) for |a| in [2^-900, 2^900] and |d| in [2^-100, 2^100] (host
// check); everything else goes through __ddiv_rn.
__device__ __forceinline__ double div_rn(double a, double d, double y) {
    const unsigned e = (static_cast<unsigned>(__double2hiint(a)) >> 20) & 0x7ffu;
    if (e - 123u < 1800u && y != 0.0) {
        const double q = __dmul_rn(a, y);
        const double r = __fma_rn(-d, q, a);
        return __fma_rn(r, y, q);
    }
    return __ddiv_rn(a, d);
}

// sum = sum + p only when pred (a predicated add: the skipped slot leaves
// every bit of sum unchanged)
__device__ __forceinline__ void add_if(double &sum, double p, bool pred) {
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q add.rn.f64 %0, %0, %1;\n}" : "+d"(sum) : "d"(p), "r"(static_cast<int>(pred)));
}

#ifndef SB_SG_MINB
#define SB_SG_MINB 4
#endif
template <int MODE, int NV, int VF, int CF, int GS, int NG>
__global__ void __launch_bounds__(kTileRows, SB_SG_MINB)
    k_sellg(int n, int nslices, const int64_t *__restrict__ soff, const unsigned char *__restrict__ blk,
            const double *__restrict__ dict, const double *__restrict__ rdict, int ndict, int ngmax,
            const double *__restrict__ x, const double *__restrict__ f, double *__restrict__ out, double omega,
            const int *skip, Aux aux, Red red) {
    constexpr int S = kSgStages;
    constexpr int H = kTileRows;
    constexpr int VB = VF ? 1 : 8, CB = CF ? 2 : 4;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[S];
    __shared__ __align__(8) uint64_t empty[S];
    __shared__ double sdict[VF ? 256 : 1];
    __shared__ double srdict[VF ? 256 : 1];
    double acc[NV > 0 ? NV : 1];
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) acc[v] = 0.0;
    const size_t sb = sg_stage_bytes(ngmax, GS, H, VF, CF);
    constexpr int kWarps = kTileRows / 32;
    const int tid = threadIdx.x;
    const bool f_al = (reinterpret_cast<uintptr_t>(f) & 15u) == 0;  // TMA needs 16-byte aligned windows

    // thread 0: stage slice t into buffer s (one bulk copy for the matrix
    // block, one for the rhs window once the predecessor is complete)
    auto issue = [&](int t, int s, bool with_f) {
        const int64_t b0 = soff[t], b1 = soff[t + 1];
        unsigned char *st = smem + s * sb;
        const int r0 = t * H;
        const int rows = min(H, n - r0);
        const uint32_t fbytes = (MODE != M_SPMV && with_f && f_al) ? static_cast<uint32_t>(rows & ~1) * 8u : 0u;
        const uint32_t mbytes = static_cast<uint32_t>(b1 - b0);
        mbar_expect_tx(&full[s], mbytes + fbytes);
        bulk_g2s(st, blk + b0, mbytes, &full[s]);
        if (fbytes) bulk_g2s(st + (sb - 8 * H), f + r0, fbytes, &full[s]);
    };

    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < S; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kWarps);
        }
        fence_mbar_init();
    }
    if constexpr (VF == 1)
        for (int i = tid; i < ndict; i += blockDim.x) {
            sdict[i] = dict[i];
            srdict[i] = rdict[i];
        }
    __syncthreads();
    const int G = static_cast<int>(gridDim.x);
    const int b = static_cast<int>(blockIdx.x);
    if (tid == 0)
        for (int q = 0; q < S - 1; ++q)
            if (b + q * G < nslices) issue(b + q * G, q, false);
    pdl_wait();
    const bool active = !(skip && *skip);
    if (!active) {
        for (int q = 0; q < S - 1; ++q)
            if (b + q * G < nslices) mbar_wait(&full[q], 0u);
        pdl_trigger();
    } else {
        uint32_t fph = 0u, eph = 0u;
        int it = 0;
        for (int t = b; t < nslices; t += G, ++it) {
            const int s = it & (S - 1);
            if (t + G >= nslices) pdl_trigger();
            const int tn = t + (S - 1) * G;
            if (tid == 0 && tn < nslices) {
                const int sn = (it + S - 1) & (S - 1);
                if (it >= 1) {
                    mbar_wait(&empty[sn], (eph >> sn) & 1u);
                    eph ^= 1u << sn;
                }
                issue(tn, sn, true);
            }
            mbar_wait(&full[s], (fph >> s) & 1u);
            fph ^= 1u << s;
            const unsigned char *st = smem + s * sb;
            const int2 gh = *reinterpret_cast<const int2 *>(st);
            const int ng = gh.x, nfull = gh.y;
            const unsigned char *sv = st + kSgHdr;
            const unsigned char *sc = sv + static_cast<size_t>(ng) * H * GS * VB;
            const uint16_t *meta = reinterpret_cast<const uint16_t *>(sc + static_cast<size_t>(ng) * H * GS * CB);
            const double *sf = reinterpret_cast<const double *>(st + (sb - 8 * H));
            const bool f_staged = it >= S - 1 && f_al;
            const int r0 = t * H;
            {
                const int lr = tid;  // row within the slice
                const int row = r0 + lr;
                if (row < n) {
                    const uint32_t m = meta[lr];
                    const int len = static_cast<int>(m & 0xffu);
                    double fi = 0.0;
                    if (MODE != M_SPMV) fi = (f_staged && lr < (min(H, n - r0) & ~1)) ? sf[lr] : f[row];
                    double xi = 0.0;
                    if constexpr (MODE >= M_JACOBI) xi = xval<MODE, false>(row, x, f, aux, omega);
                    const double *xrow = x + row;
                    double sum = 0.0;
                    // slot u of group g: value, gathered x (loads only; no arithmetic)
                    auto load = [&](int g, double *a, double *xv) {
                        using VT = typename RawVec<GS * VB>::T;
                        using CT = typename RawVec<GS * CB>::T;
                        const VT vv = *reinterpret_cast<const VT *>(sv + (static_cast<size_t>(g) * H + lr) * GS * VB);
                        const CT cc = *reinterpret_cast<const CT *>(sc + (static_cast<size_t>(g) * H + lr) * GS * CB);
#pragma unroll
                        for (int u = 0; u < GS; ++u) {
                            int col;  // CF 1: the column delta
                            if constexpr (CF == 1) {
                                const uint32_t w = word_of<GS * CB>(cc, u >> 1);
                                col = (u & 1) ? (static_cast<int>(w) >> 16) : static_cast<int>(static_cast<int16_t>(w & 0xffffu));
                            } else {
                                col = static_cast<int>(word_of<GS * CB>(cc, u));
                            }
                            if constexpr (VF == 1) {
                                const uint32_t w = word_of<GS * VB>(vv, u >> 2);
                                a[u] = sdict[(w >> (8 * (u & 3))) & 0xffu];
                            } else {
                                const uint32_t lo = word_of<GS * VB>(vv, 2 * u), hi = word_of<GS * VB>(vv, 2 * u + 1);
                                a[u] = __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
                            }
                            if constexpr (MODE == M_JACOBI || MODE == M_RESID || MODE == M_SPMV)
                                xv[u] = (CF == 1) ? __ldg(xrow + col) : __ldg(x + col);
                            else
                                xv[u] = xval<MODE, false>((CF == 1) ? row + col : col, x, f, aux, omega);
                        }
                    };
                    // sum += a*x in slot order; slots past the row length leave sum untouched
                    auto accumulate = [&](int g, const double *a, const double *xv, bool masked) {
                        if (masked) {
#pragma unroll
                            for (int u = 0; u < GS; ++u) add_if(sum, __dmul_rn(a[u], xv[u]), g * GS + u < len);
                        } else {
#pragma unroll
                            for (int u = 0; u < GS; ++u) sum = __dadd_rn(sum, __dmul_rn(a[u], xv[u]));
                        }
                    };
                    if constexpr (NG > 0) {  // compile-time group count: the gathers of 2 groups in flight at once
#pragma unroll
                        for (int g0 = 0; g0 < NG; g0 += 2) {
                            constexpr int B = 2;
                            double a[B * GS], xv[B * GS];
#pragma unroll
                            for (int q = 0; q < B; ++q)
                                if (g0 + q < NG && g0 + q < ng) load(g0 + q, a + q * GS, xv + q * GS);
#pragma unroll
                            for (int q = 0; q < B; ++q)
                                if (g0 + q < NG && g0 + q < ng) accumulate(g0 + q, a + q * GS, xv + q * GS, g0 + q >= nfull);
                        }
                    } else {
                        for (int g = 0; g < ng; ++g) {
                            double a[GS], xv[GS];
                            load(g, a, xv);
                            accumulate(g, a, xv, true);
                        }
                    }
                    double o;
                    if constexpr (MODE == M_SPMV) o = sum;
                    else if constexpr (MODE == M_RESID) o = __dsub_rn(fi, sum);
                    else {
                        double d, y;
                        const int di = static_cast<int>(m >> 8);
                        if constexpr (VF == 1) {
                            d = sdict[di];
                            y = srdict[di];
                        } else {
                            d = *reinterpret_cast<const double *>(sv + ((static_cast<size_t>(di / GS) * H + lr) * GS + (di % GS)) * 8);
                            y = 0.0;
                        }
                        o = __dadd_rn(xi, div_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), d, y));
                    }
                    out[row] = o;
                    if (NV >= 1) acc[0] += o * (red.w0 ? red.w0[row] : o);
                    if (NV >= 2) acc[NV >= 2 ? 1 : 0] += o * (red.w1 ? red.w1[row] : o);
                }
            }
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&empty[s]);
        }
    }
    if constexpr (NV > 0) finish_reduction<NV>(red, acc);
}

#include "sb_rowpat.cuh"
#include "sb_march.cuh"
#include "sb_tblock.cuh"
#include "sb_box2.cuh"

// ===========================================================================
// Cluster-resident tail: the deepest levels (each CTA's slice of every tail
// level fits in its shared memory), down to the coarsest solve and back up, in
// ONE launch of a thread-block cluster (16 CTAs where schedulable). CTA r owns
// the contiguous row block [r*rows_per, (r+1)*rows_per) of every level and
// keeps that block's CSR rows, diagonal, aggregate map, members and all level
// vectors in its shared memory; neighbour values come over DSMEM
// (ld.shared::cluster). Phases are separated by hardware cluster barriers
// (~0.2 us) instead of kernel boundaries (~2-5 us each), which is what these
// latency-bound levels pay. Arithmetic is the same bitwise row order as the
// big levels (sum = 0; sum += a*x in CSR order, no FMA).
// ===========================================================================

constexpr int kTailMaxLevels = 24;
constexpr int kTailThreads = 512;

// Per tail level, byte offsets into every CTA's shared memory (identical in
// all CTAs). The matrix part ("image") of each CTA is prepared on the host and
// arrives with ONE TMA bulk copy; the vectors follow the image.
//   ngh  int32[kTailMaxLevels] at offset 0: this CTA's ghost count per level
//   rp   int32[rows_per + 1]  local CSR offsets of the CTA's rows
//   col  uint16[nnz_cap]      column renumbered into [own rows | ghosts]
//   val  uint8 dictionary index (vf) or f64 value, per entry
//   dix  uint8 dictionary index of a_ii (vf) or f64 a_ii, per row
//   gh   uint32[gh_cap]       ghost sources: owner CTA << 16 | owner-local row,
//                             sorted by (owner, row) so pulls are coalesced
//   agg  uint32 packed coarse parent per row; mem: 2 x uint32 packed members
//        per owned coarse row (0xffffffff: none)
//   dict / rdict: the level's distinct values and their RN reciprocals
// x and t hold [own | ghost] values; a sweep first pulls its input's ghosts
// over DSMEM (only the halo crosses CTAs), then runs on local shared memory.
struct TailLevel {
    int n, rows_per, gh_cap, vf, ndict;
    int o_rp, o_col, o_val, o_dix, o_gh, o_agg, o_mem, o_dict, o_rdict;
    int o_x, o_t, o_f, o_r;
};

struct TailDesc {
    int nlev;      // including the coarsest
    int ncoarse;   // coarsest rows
    int rows_c;    // coarsest rows per CTA
    int img_bytes; // per-CTA image (multiple of 16)
    int o_inv;     // coarsest: the CTA's rows of A_c^{-1} (image)
    int o_fc;      // coarsest: gathered f_c (all rows)
    int smem_bytes;
    const unsigned char *img;  // ctas * img_bytes
    TailLevel L[kTailMaxLevels];
};

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// f64 of vector `o_vec` at packed (owner CTA << 16 | row): local shared load
// when this CTA owns it, a DSMEM load otherwise
__device__ __forceinline__ double cl_get(unsigned char *sb, uint32_t base, unsigned me, int o_vec, uint32_t e) {
    const uint32_t own = e >> 16, row = e & 0xffffu;
    if (own == me) return reinterpret_cast<const double *>(sb + o_vec)[row];
    const uint32_t a = base + static_cast<uint32_t>(o_vec) + (row << 3);
    uint32_t ra;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(own));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
    return v;
}

template <typename T> __device__ __forceinline__ T *sm(unsigned char *base, int off) {
    return reinterpret_cast<T *>(base + off);
}

// ghosts of vector o_vec (level l) <- their owners' values (after a cluster barrier)
__device__ __forceinline__ void tail_pull(unsigned char *sb, uint32_t base, unsigned me, const TailLevel &l,
                                          int ngh, int o_vec) {
    const uint32_t *gh = sm<uint32_t>(sb, l.o_gh);
    double *dst = sm<double>(sb, o_vec) + l.rows_per;
    for (int g = threadIdx.x; g < ngh; g += blockDim.x) dst[g] = cl_get(sb, base, me, o_vec, gh[g]);
    __syncthreads();
}

__device__ __forceinline__ void tail_diag(unsigned char *sb, const TailLevel &l, int li, double &d, double &y) {
    if (l.vf) {
        const int di = sm<uint8_t>(sb, l.o_dix)[li];
        d = sm<double>(sb, l.o_dict)[di];
        y = sm<double>(sb, l.o_rdict)[di];
    } else {
        d = sm<double>(sb, l.o_dix)[li];
        y = 0.0;
    }
}

// One sweep over the CTA's rows of level l (CSR order, no FMA: bitwise the
// reference's), all operands local: RESID: out = f - A x; else
// out = x + w (f - A x) / a_ii.
template <bool RESID>
__device__ __forceinline__ void tail_sweep(unsigned char *sb, const TailLevel &l, int o_in, int o_out, double omega,
                                           int m) {
    const int32_t *rp = sm<int32_t>(sb, l.o_rp);
    const uint16_t *col = sm<uint16_t>(sb, l.o_col);
    const double *xin = sm<double>(sb, o_in);
    const double *f = sm<double>(sb, l.o_f);
    const double *dict = sm<double>(sb, l.o_dict);
    for (int li = threadIdx.x; li < m; li += blockDim.x) {
        const int rs = rp[li], re = rp[li + 1];
        double sum = 0.0;
        for (int k = rs; k < re; k += 4) {
            double a[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + u < re) {
                    a[u] = l.vf ? dict[sm<uint8_t>(sb, l.o_val)[k + u]] : sm<double>(sb, l.o_val)[k + u];
                    xv[u] = xin[col[k + u]];
                }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + u < re) sum = __dadd_rn(sum, __dmul_rn(a[u], xv[u]));
        }
        if constexpr (RESID) {
            sm<double>(sb, o_out)[li] = __dsub_rn(f[li], sum);
        } else {
            double d, y;
            tail_diag(sb, l, li, d, y);
            sm<double>(sb, o_out)[li] = __dadd_rn(xin[li], div_rn(__dmul_rn(omega, __dsub_rn(f[li], sum)), d, y));
        }
    }
}

__global__ void __launch_bounds__(kTailThreads, 1)
    k_tail(const TailDesc *__restrict__ Dg, const double *f0, double *X0, double omega, int pre, int post,
           unsigned long long *trace) {
    extern __shared__ __align__(16) unsigned char sb[];
    __shared__ TailDesc D;
    __shared__ __align__(8) uint64_t bar;
    int ntr = 0;
    auto mark = [&]() {
        if (trace && threadIdx.x == 0 && cluster_rank() == 0 && ntr < 255) trace[1 + ntr++] = globaltimer();
    };
    mark();
    const unsigned me = cluster_rank();
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(TailDesc) / 4); i += blockDim.x)
        reinterpret_cast<int *>(&D)[i] = reinterpret_cast<const int *>(Dg)[i];
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // this CTA's matrix image: one bulk copy (constant data: before the dependency wait)
        mbar_expect_tx(&bar, static_cast<uint32_t>(D.img_bytes));
        bulk_g2s(sb, D.img + static_cast<size_t>(me) * D.img_bytes, static_cast<uint32_t>(D.img_bytes), &bar);
    }
    const int nlev = D.nlev;
    const uint32_t base = smem_u32(sb);
    const int *ngh = sm<int>(sb, 0);
    auto rows_of = [&](const TailLevel &l) { return max(0, min(l.rows_per, l.n - static_cast<int>(me) * l.rows_per)); };
    pdl_wait();  // the predecessor (restriction) has produced f0
    {
        const TailLevel &l = D.L[0];
        const int r0 = static_cast<int>(me) * l.rows_per, m = rows_of(l);
        for (int i = threadIdx.x; i < m; i += blockDim.x) sm<double>(sb, l.o_f)[i] = __ldcg(f0 + r0 + i);
    }
    mbar_wait(&bar, 0u);
    __syncthreads();
    mark();

    uint32_t cur_is_x = 0u;  // per level: pre-smoothed iterate in x (1) or t (0)
    // ---- down -------------------------------------------------------------------
    for (int q = 0; q + 1 < nlev; ++q) {
        const TailLevel &l = D.L[q];
        const int m = rows_of(l);
        // buffer plan: the prolongation runs in place on the pre-smoothed
        // iterate and the post-sweeps must end in x
        const int pre_end = (post % 2 == 0) ? l.o_x : l.o_t;
        int cur = pre_end;
        if (pre == 0) {
            for (int i = threadIdx.x; i < m; i += blockDim.x) sm<double>(sb, pre_end)[i] = 0.0;
        } else {
            const int first = (pre % 2 == 1) ? pre_end : (pre_end == l.o_x ? l.o_t : l.o_x);
            if (q == 0)  // deeper levels: done by the restriction
                for (int li = threadIdx.x; li < m; li += blockDim.x) {
                    double d, y;
                    tail_diag(sb, l, li, d, y);
                    sm<double>(sb, first)[li] = __dadd_rn(0.0, div_rn(__dmul_rn(omega, sm<double>(sb, l.o_f)[li]), d, y));
                }
            cur = first;
            for (int sw = 1; sw < pre; ++sw) {
                cluster_sync_all();
                mark();
                tail_pull(sb, base, me, l, ngh[q], cur);
                const int nxt = cur == l.o_x ? l.o_t : l.o_x;
                tail_sweep<false>(sb, l, cur, nxt, omega, m);
                cur = nxt;
            }
        }
        if (cur == l.o_x) cur_is_x |= 1u << q;
        cluster_sync_all();
        mark();
        tail_pull(sb, base, me, l, ngh[q], cur);
        tail_sweep<true>(sb, l, cur, l.o_r, omega, m);  // r = f - A x
        cluster_sync_all();
        mark();
        // restriction f_c = (0 + r[m0]) + r[m1]; the coarse level's first sweep rides along
        const TailLevel &lc = D.L[q + 1];
        const bool coarsest = q + 2 == nlev;
        const int mc = rows_of(lc);
        const int pe_c = (post % 2 == 0) ? lc.o_x : lc.o_t;
        const int first_c = (pre % 2 == 1) ? pe_c : (pe_c == lc.o_x ? lc.o_t : lc.o_x);
        const uint2 *mem = sm<uint2>(sb, l.o_mem);
        for (int c = threadIdx.x; c < mc; c += blockDim.x) {
            const uint2 mm = mem[c];
            double acc = __dadd_rn(0.0, cl_get(sb, base, me, l.o_r, mm.x));
            if (mm.y != 0xffffffffu) acc = __dadd_rn(acc, cl_get(sb, base, me, l.o_r, mm.y));
            sm<double>(sb, lc.o_f)[c] = acc;
            if (!coarsest && pre >= 1) {
                double d, y;
                tail_diag(sb, lc, c, d, y);
                sm<double>(sb, first_c)[c] = __dadd_rn(0.0, div_rn(__dmul_rn(omega, acc), d, y));
            }
        }
    }
    // ---- coarsest: gather f_c, own rows of A_c^{-1} f_c ------------------------------------
    {
        const TailLevel &l = D.L[nlev - 1];
        cluster_sync_all();
        mark();
        double *fc = sm<double>(sb, D.o_fc);
        for (int j = threadIdx.x; j < D.ncoarse; j += blockDim.x) {
            const uint32_t own = static_cast<uint32_t>(j / D.rows_c);
            fc[j] = cl_get(sb, base, me, l.o_f, (own << 16) | static_cast<uint32_t>(j - static_cast<int>(own) * D.rows_c));
        }
        __syncthreads();
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        const int mcr = rows_of(l);
        const double *inv = sm<double>(sb, D.o_inv);
        for (int li = warp; li < mcr; li += nw) {
            double acc = 0.0;
            for (int j = lane; j < D.ncoarse; j += 32) acc += inv[static_cast<size_t>(li) * D.ncoarse + j] * fc[j];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
            if (lane == 0) sm<double>(sb, l.o_x)[li] = acc;
        }
    }
    // ---- up -------------------------------------------------------------------------------
    for (int q = nlev - 2; q >= 0; --q) {
        const TailLevel &l = D.L[q];
        const TailLevel &lc = D.L[q + 1];
        const int m = rows_of(l);
        int cur = (cur_is_x >> q) & 1u ? l.o_x : l.o_t;
        cluster_sync_all();
        mark();
        // x += P x_c: x_i + (0.0 + x_c[agg_i]) (cycle.hpp:72-73), in place
        const uint32_t *agg = sm<uint32_t>(sb, l.o_agg);
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            double *xi = sm<double>(sb, cur) + i;
            *xi = __dadd_rn(*xi, __dadd_rn(0.0, cl_get(sb, base, me, lc.o_x, agg[i])));
        }
        for (int sw = 0; sw < post; ++sw) {
            cluster_sync_all();
            mark();
            tail_pull(sb, base, me, l, ngh[q], cur);
            const int nxt = cur == l.o_x ? l.o_t : l.o_x;
            tail_sweep<false>(sb, l, cur, nxt, omega, m);
            cur = nxt;
        }
    }
    // ---- result of tail level 0 -> X0 ------------------------------------------------------
    {
        const TailLevel &l = D.L[0];
        const int r0 = static_cast<int>(me) * l.rows_per, m = rows_of(l);
        for (int i = threadIdx.x; i < m; i += blockDim.x) X0[r0 + i] = sm<double>(sb, l.o_x)[i];
    }
    cluster_sync_all();  // no CTA exits while others may still read its shared memory
    mark();
    if (trace && threadIdx.x == 0 && cluster_rank() == 0) trace[0] = ntr;
}

// First pre-smoothing sweep from x = 0: the reference computes
// x_i = 0 + omega*(f_i - 0)/a_ii with spmv(A, 0) = +0.0 (smoother.hpp:112-119).
__global__ void k_jacobi_zero(int64_t n, const double *__restrict__ f,
                              const double *__restrict__ diag, double *__restrict__ x, double omega) {
    pdl_wait();
    pdl_trigger_single(n);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, f[i]), diag[i]));
}

// f_c[c] = (0.0 + r[m0]) + r[m1], members ascending (csr.hpp:232-239 with unit P).
// xc0 != nullptr: also the coarse level's first pre-sweep from x = 0,
// x0_c = 0 + (omega * f_c) / a_cc (smoother.hpp:112-119 with spmv(A, 0) = +0),
// so the coarse level starts at its second sweep.
__global__ void k_restrict(int64_t nc, const int2 *__restrict__ mem, const double *__restrict__ r,
                           double *__restrict__ fc, const double *__restrict__ dc, double *__restrict__ xc0,
                           double omega) {
    pdl_wait();
    pdl_trigger_single(nc);
    for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < nc;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int2 m = mem[c];
        double s = __dadd_rn(0.0, r[m.x]);
        if (m.y >= 0) s = __dadd_rn(s, r[m.y]);
        fc[c] = s;
        if (xc0) xc0[c] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, s), dc[c]));
    }
}

// out_i = in_i + (0.0 + x_c[agg_i]) (cycle.hpp:72-73: spmv(P, x_c) then axpy(1.0, ...)).
__global__ void k_prolong(int64_t n, const int32_t *__restrict__ agg, const double *xin,
                          const double *__restrict__ xc, double *xout) {
    pdl_wait();
    pdl_trigger_single(n);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        xout[i] = __dadd_rn(xin[i], __dadd_rn(0.0, xc[agg[i]]));
}

// the same, two rows per thread with 16-byte loads / stores (n even, 16-byte
// aligned vectors): the prolongation of the levels whose sweeps run as row
// pairs (k_crosspair), kept out of the first post-sweep there (emit_vcycle)
__global__ void k_prolong2(int64_t npairs, const int2 *__restrict__ agg, const double2 *xin,
                           const double *__restrict__ xc, double2 *xout) {
    pdl_wait();
    pdl_trigger_single(npairs);
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < npairs;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int2 a = agg[q];
        const double2 v = xin[q];
        const double c0 = xc[a.x], c1 = a.y == a.x ? c0 : xc[a.y];
        xout[q] = make_double2(__dadd_rn(v.x, __dadd_rn(0.0, c0)), __dadd_rn(v.y, __dadd_rn(0.0, c1)));
    }
}

// Coarsest-level solve z = A_c^{-1} f with the precomputed inverse (one warp
// per row, fixed shuffle tree).
__global__ void k_coarse_gemv(int n, const double *__restrict__ inv, const double *__restrict__ f,
                              double *__restrict__ x) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= n) return;
    const double *a = inv + static_cast<size_t>(row) * n;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += a[j] * f[j];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) x[row] = s;
}

// Bit-exact coarsest solve (parity mode): the reference's permuted forward
// substitution (column sweep keeps each row's ascending-j order) and its
// backward substitution, row by row in ascending-j order, in one thread.
// lu is the reference's row-major LU (coarse_solver.hpp:168-182).
__global__ void k_coarse_lu_exact(int n, const double *__restrict__ lu, const int32_t *__restrict__ perm,
                                  const double *__restrict__ f, double *__restrict__ x) {
    extern __shared__ double y[];
    pdl_wait();
    const int lane = threadIdx.x;
    for (int i = lane; i < n; i += 32) y[i] = f[perm[i]];
    __syncwarp();
    for (int j = 0; j < n; ++j) {
        const double yj = y[j];
        for (int i = j + 1 + lane; i < n; i += 32)
            y[i] = __dsub_rn(y[i], __dmul_rn(lu[static_cast<size_t>(i) * n + j], yj));
        __syncwarp();
    }
    if (lane == 0) {
        for (int i = n - 1; i >= 0; --i) {
            double s = y[i];
            const double *row = lu + static_cast<size_t>(i) * n;
            for (int j = i + 1; j < n; ++j) s = __dsub_rn(s, __dmul_rn(row[j], y[j]));
            y[i] = __ddiv_rn(s, row[i]);
        }
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) x[i] = y[i];
}

// ---- Krylov vector kernels (grid-stride, fixed grid => deterministic) -----

#define GRID_LOOP(i, n)                                                                          \
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (n);      \
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)

// Optional by-product of a Krylov vector kernel: the next preconditioner's
// first Jacobi sweep from 0 on level 0, x0_i = 0 + (w v_i)/a_ii for the vector
// v the kernel produces (smoother.hpp:112-119), so that V-cycle skips its
// zero-sweep kernel (harmless when the loop stops instead: x0 is unused).
struct X0 {
    const double *diag = nullptr;
    double *x0 = nullptr;
    double omega = 0.0;
    // row-pattern level 0: a_ii = pdg[pid[i]] (1 B per row instead of the 8 B
    // diagonal) and RN(1/a_ii) = pry[pid[i]] for the Markstein quotient
    const uint8_t *pid = nullptr;
    const double *pdg = nullptr, *pry = nullptr;
    __device__ __forceinline__ void put(int64_t i, double v) const {
        if (x0) x0[i] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, v), diag[i]));
    }
};

// x = 0, r = b, ||b||^2 (krylov.hpp:70-79, cycle.hpp:105-111)
__global__ void k_init(int64_t n, const double *__restrict__ b, double *__restrict__ x,
                       double *__restrict__ r, Red red) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    if (blockIdx.x == 0 && threadIdx.x == 0) red.st->t0 = globaltimer();
    double a[1] = {0.0};
    GRID_LOOP(i, n) {
        const double bi = b[i];
        x[i] = 0.0;
        if (r) r[i] = bi;
        a[0] += bi * bi;
    }
    finish_reduction<1>(red, a);
}

// Row loops of the Krylov vector kernels: two rows per step with 16-byte
// accesses when every vector is 16-byte aligned (warp-uniform test), else one.
// The per-row arithmetic is identical; only a thread's accumulation order of
// its reduction partial changes with the width (deterministic per launch).
template <int V> struct DV {
    double v[V];
};
template <int V> __device__ __forceinline__ DV<V> ldv(const double *p, int64_t i) {
    DV<V> o;
    if constexpr (V == 2) {
        const double2 t = *reinterpret_cast<const double2 *>(p + i);
        o.v[0] = t.x;
        o.v[1] = t.y;
    } else {
        o.v[0] = p[i];
    }
    return o;
}
template <int V> __device__ __forceinline__ void stv(double *p, int64_t i, const DV<V> &x) {
    if constexpr (V == 2) *reinterpret_cast<double2 *>(p + i) = make_double2(x.v[0], x.v[1]);
    else p[i] = x.v[0];
}
__device__ __forceinline__ bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
template <typename... P> __device__ __forceinline__ bool all16(const P *...p) { return (al16(p) && ...); }
template <typename Body> __device__ __forceinline__ void grid_rows(int64_t n, bool vec, Body &&body) {
    if (vec) {
        const int64_t h = n / 2;
        GRID_LOOP(q, h) body(std::integral_constant<int, 2>{}, 2 * q);
        if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) body(std::integral_constant<int, 1>{}, n - 1);
    } else {
        GRID_LOOP(i, n) body(std::integral_constant<int, 1>{}, i);
    }
}
__device__ __forceinline__ bool x0_ok(const X0 &z0) {
    return !z0.x0 || (al16(z0.x0) && (z0.pid || al16(z0.diag)));
}
template <int V> __device__ __forceinline__ void x0_put(const X0 &z0, int64_t i, const DV<V> &v) {
    if (!z0.x0) return;
    DV<V> o;
    if (z0.pid) {  // table a_ii and its reciprocal: div_rn is the IEEE quotient (its range checks fall back)
        int p[V];
        if constexpr (V == 2) {
            const uint32_t pp = *reinterpret_cast<const uint16_t *>(z0.pid + i);
            p[0] = pp & 0xff;
            p[V - 1] = pp >> 8;
        } else {
            p[0] = z0.pid[i];
        }
#pragma unroll
        for (int k = 0; k < V; ++k)
            o.v[k] = __dadd_rn(0.0, div_rn(__dmul_rn(z0.omega, v.v[k]), __ldg(z0.pdg + p[k]), __ldg(z0.pry + p[k])));
    } else {
        const DV<V> d = ldv<V>(z0.diag, i);
#pragma unroll
        for (int k = 0; k < V; ++k) o.v[k] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(z0.omega, v.v[k]), d.v[k]));
    }
    stv<V>(z0.x0, i, o);
}

// dst = src; sum src*w  (PCG: p = z, rz = (r, z); BiCGStab: rbar = p = r, rho = (r, rbar))
__global__ void k_copy_dot(int64_t n, const double *__restrict__ src, double *__restrict__ dst,
                           double *__restrict__ dst2, const double *__restrict__ w, Red red, X0 z0) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    double a[1] = {0.0};
    grid_rows(n, all16(src, dst, w) && (!dst2 || al16(dst2)) && x0_ok(z0), [&](auto vc, int64_t i) {
        constexpr int V = decltype(vc)::value;
        const DV<V> sv = ldv<V>(src, i), wv = ldv<V>(w, i);
        stv<V>(dst, i, sv);
        if (dst2) stv<V>(dst2, i, sv);
#pragma unroll
        for (int k = 0; k < V; ++k) a[0] += sv.v[k] * wv.v[k];
        x0_put<V>(z0, i, sv);
    });
    finish_reduction<1>(red, a);
}
__global__ void k_dot(int64_t n, const double *__restrict__ u, const double *__restrict__ v,
                      const int *skip, Red red) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    double a[1] = {0.0};
    if (!(skip && *skip)) {
        grid_rows(n, all16(u, v), [&](auto vc, int64_t i) {
            constexpr int V = decltype(vc)::value;
            const DV<V> uv = ldv<V>(u, i), vv = ldv<V>(v, i);
#pragma unroll
            for (int k = 0; k < V; ++k) a[0] += uv.v[k] * vv.v[k];
        });
    }
    finish_reduction<1>(red, a);
}
// PCG update (krylov.hpp:96-98): x += alpha p; r += (-alpha) Ap; ||r||^2 (+ x0 of z = M r)
__global__ void k_pcg_update(int64_t n, double *__restrict__ x, double *__restrict__ r,
                             const double *__restrict__ p, const double *__restrict__ Ap, Red red, X0 z0) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    double a[1] = {0.0};
    const DevState *st = red.st;
    if (!st->done) {
        const double alpha = st->alpha, nalpha = -st->alpha;
        grid_rows(n, all16(x, r, p, Ap) && x0_ok(z0), [&](auto vc, int64_t i) {
            constexpr int V = decltype(vc)::value;
            DV<V> xv = ldv<V>(x, i), rv = ldv<V>(r, i);
            const DV<V> pv = ldv<V>(p, i), av = ldv<V>(Ap, i);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                xv.v[k] = __dadd_rn(xv.v[k], __dmul_rn(alpha, pv.v[k]));
                rv.v[k] = __dadd_rn(rv.v[k], __dmul_rn(nalpha, av.v[k]));
                a[0] += rv.v[k] * rv.v[k];
            }
            stv<V>(x, i, xv);
            stv<V>(r, i, rv);
            x0_put<V>(z0, i, rv);
        });
    }
    finish_reduction<1>(red, a);
}
// PCG with the x update deferred (single-GPU graph): r += (-alpha) Ap; ||r||^2
// (+ x0 of z = M r). x += alpha p is applied by the next k_xpay_x (which reads
// p anyway) or, when the loop stops here, by k_x_final: the same operation on
// the same values, so x is bit for bit krylov.hpp:96-97's; the update kernel
// no longer streams x and p (16 B/row less per iteration, 8 B/row net).
__global__ void k_pcg_update_r(int64_t n, double *__restrict__ r, const double *__restrict__ Ap, Red red, X0 z0) {
    pdl_wait();
    pdl_trigger_single(n);
    double a[1] = {0.0};
    DevState *st = red.st;
    if (!st->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->x_pending = 1;
        const double nalpha = -st->alpha;
        grid_rows(n, all16(r, Ap) && x0_ok(z0), [&](auto vc, int64_t i) {
            constexpr int V = decltype(vc)::value;
            DV<V> rv = ldv<V>(r, i);
            const DV<V> av = ldv<V>(Ap, i);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                rv.v[k] = __dadd_rn(rv.v[k], __dmul_rn(nalpha, av.v[k]));
                a[0] += rv.v[k] * rv.v[k];
            }
            stv<V>(r, i, rv);
            x0_put<V>(z0, i, rv);
        });
    }
    finish_reduction<1>(red, a);
}
// x += alpha p (the deferred update, krylov.hpp:96), then p = z + beta p (krylov.hpp:113)
__global__ void k_xpay_x(int64_t n, const double *__restrict__ z, double *__restrict__ p, double *__restrict__ x,
                         DevState *__restrict__ st) {
    pdl_wait();
    pdl_trigger_single(n);
    const double beta = st->beta, alpha = st->alpha;
    grid_rows(n, all16(z, p, x), [&](auto vc, int64_t i) {
        constexpr int V = decltype(vc)::value;
        const DV<V> zv = ldv<V>(z, i);
        DV<V> pv = ldv<V>(p, i), xv = ldv<V>(x, i);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            xv.v[k] = __dadd_rn(xv.v[k], __dmul_rn(alpha, pv.v[k]));
            pv.v[k] = __dadd_rn(zv.v[k], __dmul_rn(beta, pv.v[k]));
        }
        stv<V>(x, i, xv);
        stv<V>(p, i, pv);
    });
    if (blockIdx.x == 0 && threadIdx.x == 0) st->x_pending = 0;
}
// the last iteration's deferred x += alpha p (if its update kernel ran)
__global__ void k_x_final(int64_t n, double *__restrict__ x, const double *__restrict__ p,
                          DevState *__restrict__ st) {
    pdl_wait();
    pdl_trigger_single(n);
    if (!st->x_pending) return;
    const double alpha = st->alpha;
    grid_rows(n, all16(x, p), [&](auto vc, int64_t i) {
        constexpr int V = decltype(vc)::value;
        DV<V> xv = ldv<V>(x, i);
        const DV<V> pv = ldv<V>(p, i);
#pragma unroll
        for (int k = 0; k < V; ++k) xv.v[k] = __dadd_rn(xv.v[k], __dmul_rn(alpha, pv.v[k]));
        stv<V>(x, i, xv);
    });
}
// p = z + beta p (krylov.hpp:113)
__global__ void k_xpay(int64_t n, const double *__restrict__ z, double *__restrict__ p,
                       const DevState *__restrict__ st) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    const double beta = st->beta;
    grid_rows(n, all16(z, p), [&](auto vc, int64_t i) {
        constexpr int V = decltype(vc)::value;
        const DV<V> zv = ldv<V>(z, i);
        DV<V> pv = ldv<V>(p, i);
#pragma unroll
        for (int k = 0; k < V; ++k) pv.v[k] = __dadd_rn(zv.v[k], __dmul_rn(beta, pv.v[k]));
        stv<V>(p, i, pv);
    });
}
// BiCGStab s = r + (-alpha) Ap~; ||s||^2 (krylov.hpp:164-166)
__global__ void k_bi_s(int64_t n, const double *__restrict__ r, const double *__restrict__ Apt,
                       double *__restrict__ s, Red red, X0 z0) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    double a[1] = {0.0};
    const DevState *st = red.st;
    if (!st->done) {
        const double nalpha = -st->alpha;
        grid_rows(n, all16(r, Apt, s) && x0_ok(z0), [&](auto vc, int64_t i) {
            constexpr int V = decltype(vc)::value;
            const DV<V> rv = ldv<V>(r, i), av = ldv<V>(Apt, i);
            DV<V> sv;
#pragma unroll
            for (int k = 0; k < V; ++k) {
                sv.v[k] = __dadd_rn(rv.v[k], __dmul_rn(nalpha, av.v[k]));
                a[0] += sv.v[k] * sv.v[k];
            }
            stv<V>(s, i, sv);
            x0_put<V>(z0, i, sv);
        });
    }
    finish_reduction<1>(red, a);
}
// Half-step exit: x += alpha p~ (krylov.hpp:168), only when EP_BI_SN fired.
__global__ void k_bi_half(int64_t n, double *__restrict__ x, const double *__restrict__ pt,
                          const DevState *__restrict__ st) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    if (!st->half) return;
    const double alpha = st->alpha;
    grid_rows(n, all16(x, pt), [&](auto vc, int64_t i) {
        constexpr int V = decltype(vc)::value;
        DV<V> xv = ldv<V>(x, i);
        const DV<V> pv = ldv<V>(pt, i);
#pragma unroll
        for (int k = 0; k < V; ++k) xv.v[k] = __dadd_rn(xv.v[k], __dmul_rn(alpha, pv.v[k]));
        stv<V>(x, i, xv);
    });
}
// x += alpha p~; x += omega s~; r = s + (-omega) As~; ||r||^2, (r, rbar0)  (krylov.hpp:182-186, 201)
__global__ void k_bi_update(int64_t n, double *__restrict__ x, double *__restrict__ r,
                            const double *__restrict__ pt, const double *__restrict__ st_,
                            const double *__restrict__ s, const double *__restrict__ Ast,
                            const double *__restrict__ rbar, Red red) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    double a[2] = {0.0, 0.0};
    const DevState *st = red.st;
    if (!st->done) {
        const double alpha = st->alpha, omega = st->omega, nomega = -st->omega;
        grid_rows(n, all16(x, r, pt, st_, s, Ast, rbar), [&](auto vc, int64_t i) {
            constexpr int V = decltype(vc)::value;
            DV<V> xv = ldv<V>(x, i), rv;
            const DV<V> pv = ldv<V>(pt, i), tv = ldv<V>(st_, i), sv = ldv<V>(s, i), av = ldv<V>(Ast, i),
                        bv = ldv<V>(rbar, i);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const double xi = __dadd_rn(xv.v[k], __dmul_rn(alpha, pv.v[k]));
                xv.v[k] = __dadd_rn(xi, __dmul_rn(omega, tv.v[k]));
                rv.v[k] = __dadd_rn(sv.v[k], __dmul_rn(nomega, av.v[k]));
                a[0] += rv.v[k] * rv.v[k];
                a[1] += rv.v[k] * bv.v[k];
            }
            stv<V>(x, i, xv);
            stv<V>(r, i, rv);
        });
    }
    finish_reduction<2>(red, a);
}
// p = r + beta (p - omega Ap~)  (krylov.hpp:204-205)
__global__ void k_bi_p(int64_t n, const double *__restrict__ r, double *__restrict__ p,
                       const double *__restrict__ Apt, const DevState *__restrict__ st, X0 z0) {
    pdl_wait();  // launched with PDL on the partitioned path
    pdl_trigger_single(n);
    if (st->done) return;
    const double beta = st->beta, omega = st->omega;
    grid_rows(n, all16(r, p, Apt) && x0_ok(z0), [&](auto vc, int64_t i) {
        constexpr int V = decltype(vc)::value;
        const DV<V> rv = ldv<V>(r, i), av = ldv<V>(Apt, i);
        DV<V> pv = ldv<V>(p, i);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            pv.v[k] = __dadd_rn(rv.v[k], __dmul_rn(beta, __dsub_rn(pv.v[k], __dmul_rn(omega, av.v[k]))));
        }
        stv<V>(p, i, pv);
        x0_put<V>(z0, i, pv);
    });
}
__global__ void k_fill(int64_t n, double *x, double v) {
    pdl_wait();  // launched with PDL on the partitioned path
    GRID_LOOP(i, n) x[i] = v;
}

__global__ void k_set_cond(const DevState *st, CondSet cs) {
    pdl_wait();  // launched with PDL on the partitioned path
    for (int i = 0; i < cs.n; ++i)
        cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(cs.h[i]), st->done ? 0u : 1u);
}

// ===========================================================================
// device hierarchy + context
// ===========================================================================

struct DevLevel {
    int64_t n = 0, nnz = 0, nc = -1;
    int32_t *rp = nullptr, *ci = nullptr, *agg = nullptr, *tiles = nullptr;
    double *v = nullptr, *diag = nullptr;
    // streamed storage format (see Ent<>): vf 1 = uint8 dictionary values,
    // cf 1 = int16 column deltas; the raw ci / v stay for the cluster tail
    int vf = 0, cf = 0, ndict = 0;
    const void *sv = nullptr, *sc = nullptr;
    double *dict = nullptr;
    // grouped sliced-ELL layout (sell = 1): byte offsets of the slice blocks,
    // the blocks, the reciprocal dictionary (Markstein division)
    int sell = 0, sell_tiles = 0, sell_ngmax = 0, sell_gs = 4, sell_grid = 0;
    size_t sell_smem = 0;
    int64_t *soff = nullptr;
    const unsigned char *sell_blk = nullptr;
    int64_t sell_slots = 0;  // stored entry slots (incl. padding)
    double *rdict = nullptr;
    // row-pattern layout (pat = 1): one pattern index per row + the pattern table
    int pat = 0, pat_np = 0, pat_w = 0, pat_grid = 0;
    // the most frequent pattern (k_rowpat's MainPat parameter): id, len, a_ii,
    // RN(1/a_ii), values and offsets (W slots, padding included)
    int main_p = -1, main_len = 0;
    double main_d = 0.0, main_r = 0.0;
    std::vector<double> main_v;
    std::vector<int> main_o;
    size_t pat_tb = 0;
    // marching sweep (k_march, sb_march.cuh): geometry of the main pattern
    // (-1: none), march stride, offset range, table, tiles of 32 rows x K steps
    int march_geo = -1, march_S = 0, march_N = 0, march_nqf = 0, march_nxb = 0, march_nyb = 0, march_ntiles = 0;
    int march_grid = 0;
    size_t march_tb = 0;
    // two fused Jacobi sweeps per launch on mid-size structured 7-point levels
    // (k_cross_box2; tb = 2) or per HBM pass (experimental k_cross_tb2; tb = 1)
    int tb = 0, tb_grid = 0, box_tx = 0;
    BoxGeo box_geo{};
    TbGeo tb_geo{};
    size_t tb_smem = 0;
    const double *tb_tab = nullptr;
    // row pairs on 27-point box levels with even strides (k_boxpair)
    int box_pair = 0, box_grid = 0, box_grid_nv = 0;  // box_grid_nv: the fused-dot variants
    const uint32_t *box_rmask = nullptr;
    const unsigned char *march_table = nullptr;
    const uint8_t *pat_id = nullptr;
    const unsigned char *pat_table = nullptr;
    int2 *mem = nullptr;
    bool pair_aggs = false;  // mem[c] == (2c, 2c + 1) for every coarse row
    int ntiles = 0, cap = 0, grid = 0;
    size_t smem = 0;
    double *x = nullptr, *f = nullptr, *t = nullptr;
    int64_t bad_diag = -1;
};

struct Cyc {
    int pre = 6, post = 6;
    double omega = 2.0 / 3.0;
};

// Kernels a whole-solve graph executes: pre + once (prologue body, when the
// loop is entered) + iterations x per_it + (iterations - skipped) x per_it_cond
// + post. Counted while the graph is captured (launch_count deltas).
struct LaunchPlan {
    int pre = 0, once = 0, per_it = 0, per_it_cond = 0, post = 0;
};

struct GraphEntry {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    LaunchPlan plan;
};

} // namespace sb

struct sb_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t cap[8] = {};
    std::vector<sb::DevLevel> L;
    int64_t nc = 0;
    double *inv = nullptr;
    double *lu = nullptr;
    int32_t *perm = nullptr;
    bool coarse_exact = false;
    double *rs = nullptr;  // residual scratch (level sizes <= n0)
    double *kv[12] = {};   // Krylov vectors
    double *partials = nullptr;
    unsigned *counter = nullptr;
    sb::DevState *st = nullptr;
    double *hist_r = nullptr, *hist_t = nullptr;
    int hist_cap = 0;
    int64_t bytes = 0;
    int nvec_blocks = 1;
    bool graphs = true;
    sb::LaunchPlan plan;         // of the graph being built
    std::map<std::tuple<const void *, int, int, int, int, int>, CUtensorMap> tmaps;  // TMA descriptors by (ptr, dims, box)
    int64_t last_launches = 0;   // kernels the last solve executed
    std::vector<void *> allocs;
    std::vector<void *> host_allocs;  // hybrid mode: pinned mapped host arrays
    bool alloc_host = false;
    int64_t host_bytes = 0;
    int host_from = 1 << 30;          // first host-resident level (hybrid mode)
    std::map<std::string, sb::GraphEntry> cache;
    double *h_pinned = nullptr;  // staging for host vectors
    int64_t h_pinned_n = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_solve_ms = 0.0;
    int tail_from = 1 << 30;  // first level run inside the cluster tail kernel
    int tail_ctas = 0;
    int tail_smem = 0;
    int tail_min = 0;  // the tail never starts above this level (partitioned levels)
    unsigned long long *trace = nullptr;  // SB_TAIL_TRACE=1: per-phase timestamps of the tail
    bool pdl = true;                      // programmatic dependent launch in the V-cycle (SB_PDL=0 off)
    sb::TailDesc *tail = nullptr;
    int launch_count = 0;  // kernels emitted by the last emit_* sequence
    // PCG: the V-cycle's last level-0 post-sweep also reduces (z, f) = (z, r)
    // into this reduction (no separate dot kernel); cleared once emitted
    const sb::Red *final_red = nullptr;
    bool final_red_used = false;
};

namespace sb {

enum KV { KX = 0, KR, KZ, KP, KAP, KRBAR, KPT, KAPT, KS, KST, KAST, KB };

// Device allocation (zeroed). While c->alloc_host is set (hybrid mode, levels
// >= host_levels_from) the arrays live in pinned, mapped host memory instead:
// the same kernels read them over the host link (zero-copy), and they do not
// count toward the device-resident bytes.
template <typename T> static T *dalloc(sb_ctx c, int64_t count, bool track = true) {
    void *p = nullptr;
    const size_t bytes = sizeof(T) * static_cast<size_t>(std::max<int64_t>(count, 1));
    if (c->alloc_host) {
        CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        std::memset(p, 0, bytes);
        c->host_allocs.push_back(p);
        if (track) c->host_bytes += static_cast<int64_t>(bytes);
        return static_cast<T *>(p);
    }
    CK(cudaMalloc(&p, bytes));
    CK(cudaMemset(p, 0, bytes));
    c->allocs.push_back(p);
    if (track) c->bytes += static_cast<int64_t>(bytes);
    return static_cast<T *>(p);
}

static int vec_grid(int64_t n) {
    const int64_t b = (n + kVecThreads - 1) / kVecThreads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8)));
}

static Red make_red(sb_ctx c, int op, int nval, const double *w0 = nullptr, const double *w1 = nullptr,
                    CondSet cs = {{0, 0}, 0}) {
    Red r;
    r.partials = c->partials;
    r.counter = c->counter;
    r.st = c->st;
    r.op = op;
    r.nval = nval;
    r.w0 = w0;
    r.w1 = w1;
    r.cs = cs;
    return r;
}

// Eager mode (sb_device_opts.use_graphs = 0): the solve drivers below emit the
// same kernels straight onto the stream and the host evaluates each
// conditional node itself (every condition in this file is !st->done).
static thread_local bool tl_eager = false;

static CondSet conds(std::initializer_list<cudaGraphConditionalHandle> hs) {
    CondSet cs{{0, 0}, 0};
    if (tl_eager) return cs;
    for (auto h : hs) cs.h[cs.n++] = static_cast<unsigned long long>(h);
    return cs;
}

// ---- launchers (each counts the kernels it emits) -------------------------------

static const bool c_pair_rr_off = [] {  // SB_PAIR_RR=0: k_pat_resid_restrict on pair levels too
    const char *e = std::getenv("SB_PAIR_RR");
    return e && std::atoi(e) == 0;
}();
static const bool c_cross_rr_off = [] {  // opt-in (SB_CROSS_RR=1): measured slower than k_pat_resid_restrict
    const char *e = std::getenv("SB_CROSS_RR");   // (C2 14.07 vs 13.70 ms, T256 98.0 vs 97.6 ms)
    return !(e && std::atoi(e) != 0);
}();

static const bool c_main_off = [] {  // SB_MAIN_PAT=0: every warp reads the shared-memory table (A/B only)
    const char *e = std::getenv("SB_MAIN_PAT");
    return e && std::atoi(e) == 0;
}();

// Launch with programmatic dependent launch (the kernel calls pdl_wait()
// before touching its predecessor's outputs) when the context enables it.
template <typename... KArgs, typename... Args>
static void launch_k(sb_ctx c, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args &&...args) {
    ++c->launch_count;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = c->pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

template <int MODE, int NV, int VF, int CF>
static void launch_csr_f(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *x, const double *f,
                         double *out, double omega, const int *skip, const Red &red, Aux aux) {
    launch_k(c, k_csr_tile<MODE, NV, VF, CF>, dim3(std::min(l.ntiles, l.grid)), dim3(kTileRows), l.smem, s,
             static_cast<const int32_t *>(l.rp), l.sc, l.sv, static_cast<const double *>(l.dict), l.ndict,
             static_cast<const int32_t *>(l.tiles), static_cast<int>(l.ntiles), x, f, out, omega, l.cap, skip, aux,
             red);
}

template <int MODE, int NV, int VF, int CF, int GS, int NG>
static void launch_sell_g(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *x, const double *f,
                          double *out, double omega, const int *skip, const Red &red, Aux aux) {
    launch_k(c, k_sellg<MODE, NV, VF, CF, GS, NG>, dim3(std::min(l.sell_tiles, l.sell_grid)), dim3(kTileRows),
             l.sell_smem, s, static_cast<int>(l.n), l.sell_tiles, static_cast<const int64_t *>(l.soff), l.sell_blk,
             static_cast<const double *>(l.dict), static_cast<const double *>(l.rdict), l.ndict, l.sell_ngmax, x, f,
             out, omega, skip, aux, red);
}

// The fast format (dictionary values, int16 deltas, groups of 4) gets a
// compile-time group count up to 7 (w <= 28: every 2D/3D 5/7/9/27-point
// stencil level); everything else runs the runtime group loop.
template <int MODE, int NV, int VF, int CF>
static void launch_sell_f(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *x, const double *f,
                          double *out, double omega, const int *skip, const Red &red, Aux aux) {
    if (l.sell_gs == 4) {
        if constexpr (VF == 1 && CF == 1) {
            switch (l.sell_ngmax) {
            case 1: return launch_sell_g<MODE, NV, 1, 1, 4, 1>(c, l, s, x, f, out, omega, skip, red, aux);
            case 2: return launch_sell_g<MODE, NV, 1, 1, 4, 2>(c, l, s, x, f, out, omega, skip, red, aux);
            case 3: return launch_sell_g<MODE, NV, 1, 1, 4, 3>(c, l, s, x, f, out, omega, skip, red, aux);
            case 4: return launch_sell_g<MODE, NV, 1, 1, 4, 4>(c, l, s, x, f, out, omega, skip, red, aux);
            case 5: return launch_sell_g<MODE, NV, 1, 1, 4, 5>(c, l, s, x, f, out, omega, skip, red, aux);
            case 6: return launch_sell_g<MODE, NV, 1, 1, 4, 6>(c, l, s, x, f, out, omega, skip, red, aux);
            case 7: return launch_sell_g<MODE, NV, 1, 1, 4, 7>(c, l, s, x, f, out, omega, skip, red, aux);
            default: break;
            }
        }
        launch_sell_g<MODE, NV, VF, CF, 4, 0>(c, l, s, x, f, out, omega, skip, red, aux);
    } else {
        launch_sell_g<MODE, NV, VF, CF, 2, 0>(c, l, s, x, f, out, omega, skip, red, aux);
    }
}

template <int W> static MainPat<W> main_pat(const DevLevel &l) {
    MainPat<W> m;
    std::memset(&m, 0, sizeof(m));
    m.p = c_main_off ? -1 : l.main_p;
    m.len = l.main_len;
    m.d = l.main_d;
    m.r = l.main_r;
    for (int k = 0; k < W && k < static_cast<int>(l.main_v.size()); ++k) {
        m.v[k] = l.main_v[static_cast<size_t>(k)];
        m.o[k] = l.main_o[static_cast<size_t>(k)];
    }
    return m;
}

template <int MODE, int NV, int W>
static void launch_pat_w(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *x, const double *f,
                         double *out, double omega, const int *skip, const Red &red, Aux aux) {
    launch_k(c, k_rowpat<MODE, NV, W>, dim3(l.pat_grid), dim3(kPatThreads), l.pat_tb, s, static_cast<int>(l.n),
             l.pat_id, l.pat_np, l.pat_table, main_pat<W>(l), x, f, out, omega, skip, aux, red);
}

template <int MODE, int NV, int G, int WP>
static void launch_march_g(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *x, const double *f,
                           double *out, double omega, const int *skip, const Red &red) {
    MarchPat<Geo<G>::W> m;
    std::memset(&m, 0, sizeof(m));
    for (int k = 0; k < Geo<G>::W; ++k) m.v[k] = l.main_v[static_cast<size_t>(k)];
    m.d = l.main_d;
    m.r = l.main_r;
    m.p = c_main_off ? -1 : l.main_p;
    m.P = l.march_S;
    m.N = l.march_N;
    m.NY = l.march_S / l.march_N;
    m.nqf = l.march_nqf;
    m.nxb = l.march_nxb;
    m.nyb = l.march_nyb;
    m.ntiles = l.march_ntiles;
    auto kern = ((l.march_S | l.march_N) & 1) ? k_march<MODE, NV, G, WP, false> : k_march<MODE, NV, G, WP, true>;
    launch_k(c, kern, dim3(l.march_grid), dim3(kMarchThreads), march_smem_bytes(l.pat_tb, l.march_tb), s, static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table,
             static_cast<int>(l.pat_tb), l.march_table, static_cast<int>(l.march_tb), m, x, f, out, omega, skip, red);
}

template <int MODE, int NV>
static void launch_csr(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *x, const double *f,
                       double *out, double omega, const int *skip, const Red &red, Aux aux = Aux{}) {
    if (l.n == 0) return;
    if constexpr (MODE == M_JACOBI || MODE == M_SPMV || MODE == M_RESID) {
        auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        if (l.pat && l.box_pair && a16(x) && a16(out) && (MODE == M_SPMV || a16(f))) {
            if (l.box_pair == 1)
                launch_k(c, k_boxpair<MODE, NV>, dim3(l.box_grid), dim3(kBoxThreads), l.pat_tb, s,
                         static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<28>(l), x, f,
                         out, omega, skip, red);
            else if (l.pat_w == 7)
                launch_k(c, k_crosspair<MODE, NV, 7>, dim3(NV > 0 ? l.box_grid_nv : l.box_grid), dim3(kCrossThreads), l.pat_tb, s,
                         static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<7>(l), x, f,
                         out, omega, skip, red, 0, static_cast<int>(l.n / 2));
            else
                launch_k(c, k_crosspair<MODE, NV, 5>, dim3(NV > 0 ? l.box_grid_nv : l.box_grid), dim3(kCrossThreads), l.pat_tb, s,
                         static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<5>(l), x, f,
                         out, omega, skip, red, 0, static_cast<int>(l.n / 2));
            return;
        }
        if constexpr (kExperimental)
            if (l.pat && l.march_geo >= 0) return launch_march_g<MODE, NV, 0, 28>(c, l, s, x, f, out, omega, skip, red);
    }
    if constexpr (MODE == M_JACOBI_PROLONG && NV == 0) {
        // aggregates = row pairs: k_crosspair with x' = x + (0 + x_c[j / 2]) at its reads (x_c in red.w0)
        auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        if (l.pat && l.box_pair == 2 && l.pair_aggs && a16(x) && a16(out) && a16(f)) {
            Red rx{};
            rx.w0 = aux.xc;
            if (l.pat_w == 7)
                launch_k(c, k_crosspair<MODE, 0, 7>, dim3(l.box_grid), dim3(kCrossThreads), l.pat_tb, s,
                         static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<7>(l), x, f,
                         out, omega, skip, rx, 0, static_cast<int>(l.n / 2));
            else
                launch_k(c, k_crosspair<MODE, 0, 5>, dim3(l.box_grid), dim3(kCrossThreads), l.pat_tb, s,
                         static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<5>(l), x, f,
                         out, omega, skip, rx, 0, static_cast<int>(l.n / 2));
            return;
        }
    }
    if (l.pat) {
        switch (l.pat_w) {
        case 5: return launch_pat_w<MODE, NV, 5>(c, l, s, x, f, out, omega, skip, red, aux);
        case 7: return launch_pat_w<MODE, NV, 7>(c, l, s, x, f, out, omega, skip, red, aux);
        case 8: return launch_pat_w<MODE, NV, 8>(c, l, s, x, f, out, omega, skip, red, aux);
        case 16: return launch_pat_w<MODE, NV, 16>(c, l, s, x, f, out, omega, skip, red, aux);
        case 28: return launch_pat_w<MODE, NV, 28>(c, l, s, x, f, out, omega, skip, red, aux);
        default: return launch_pat_w<MODE, NV, 32>(c, l, s, x, f, out, omega, skip, red, aux);
        }
    }
    if (l.sell) {
        if (l.vf && l.cf) launch_sell_f<MODE, NV, 1, 1>(c, l, s, x, f, out, omega, skip, red, aux);
        else if (l.vf) launch_sell_f<MODE, NV, 1, 0>(c, l, s, x, f, out, omega, skip, red, aux);
        else if (l.cf) launch_sell_f<MODE, NV, 0, 1>(c, l, s, x, f, out, omega, skip, red, aux);
        else launch_sell_f<MODE, NV, 0, 0>(c, l, s, x, f, out, omega, skip, red, aux);
        return;
    }
    if (l.vf && l.cf) launch_csr_f<MODE, NV, 1, 1>(c, l, s, x, f, out, omega, skip, red, aux);
    else if (l.vf) launch_csr_f<MODE, NV, 1, 0>(c, l, s, x, f, out, omega, skip, red, aux);
    else if (l.cf) launch_csr_f<MODE, NV, 0, 1>(c, l, s, x, f, out, omega, skip, red, aux);
    else launch_csr_f<MODE, NV, 0, 0>(c, l, s, x, f, out, omega, skip, red, aux);
}

template <int W>
static void launch_pat_rr_w(sb_ctx c, const DevLevel &l, const DevLevel &lc, cudaStream_t s, const double *x,
                            const double *f, double *x0, double omega) {
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((lc.n + kPatThreads - 1) / kPatThreads,
                                                                             static_cast<int64_t>(l.pat_grid) * 2)));
    launch_k(c, k_pat_resid_restrict<W>, dim3(grid), dim3(kPatThreads), l.pat_tb, s, static_cast<int>(lc.n),
             static_cast<const int2 *>(l.mem), l.pat_id, l.pat_np, l.pat_table, x, f, lc.f,
             static_cast<const double *>(lc.diag), x0, omega);
}

static void launch_pat_rr(sb_ctx c, const DevLevel &l, const DevLevel &lc, cudaStream_t s, const double *x,
                          const double *f, double *x0, double omega) {
    auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (l.box_pair == 2 && l.pair_aggs && a16(x) && a16(f) && !c_pair_rr_off) {
        // k_crosspair computes both rows of coarse row q; the coarse diagonal and
        // the first-sweep destination travel in the (otherwise unused) Red slots
        Red rr{};
        rr.w0 = lc.diag;
        rr.w1 = x0;
        if (lc.pat && lc.pat_np > 0) {
            rr.pid = lc.pat_id;
            rr.pdg = reinterpret_cast<const double *>(lc.pat_table) + static_cast<size_t>(lc.pat_np) * ((lc.pat_w + 1) & ~1);
        }
        if (l.pat_w == 7)
            launch_k(c, k_crosspair<M_RESID_RESTRICT, 0, 7>, dim3(l.box_grid), dim3(kCrossThreads), l.pat_tb, s,
                     static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<7>(l), x, f, lc.f,
                     omega, static_cast<const int *>(nullptr), rr, 0, static_cast<int>(l.n / 2));
        else
            launch_k(c, k_crosspair<M_RESID_RESTRICT, 0, 5>, dim3(l.box_grid), dim3(kCrossThreads), l.pat_tb, s,
                     static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<5>(l), x, f, lc.f,
                     omega, static_cast<const int *>(nullptr), rr, 0, static_cast<int>(l.n / 2));
        return;
    }
#if SB_EXPERIMENTAL
    if (l.box_pair == 2 && l.pat_w == 7 && a16(x) && a16(f) && !c_cross_rr_off) {
        const int grid = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>((lc.n + kCrossThreads - 1) / kCrossThreads, static_cast<int64_t>(l.box_grid))));
        launch_k(c, k_cross_rr<7>, dim3(grid), dim3(kCrossThreads), l.pat_tb, s, static_cast<int>(lc.n),
                 static_cast<const int2 *>(l.mem), static_cast<int>(l.n), l.pat_id, l.pat_np, l.pat_table, l.box_rmask,
                 main_pat<7>(l), x, f, lc.f, static_cast<const double *>(lc.diag), x0, omega);
        return;
    }
#else
    (void)a16;
#endif
    switch (l.pat_w) {
    case 5: return launch_pat_rr_w<5>(c, l, lc, s, x, f, x0, omega);
    case 7: return launch_pat_rr_w<7>(c, l, lc, s, x, f, x0, omega);
    case 8: return launch_pat_rr_w<8>(c, l, lc, s, x, f, x0, omega);
    case 16: return launch_pat_rr_w<16>(c, l, lc, s, x, f, x0, omega);
    case 28: return launch_pat_rr_w<28>(c, l, lc, s, x, f, x0, omega);
    default: return launch_pat_rr_w<32>(c, l, lc, s, x, f, x0, omega);
    }
}

static void launch_jacobi(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *xin, const double *f,
                          double *xout, double omega) {
    launch_csr<M_JACOBI, 0>(c, l, s, xin, f, xout, omega, nullptr, Red{});
}

// A Jacobi sweep over the row pairs [q_lo, q_hi) of a k_crosspair level (the
// partitioned path: interior while the halo is in flight, then the edges).
static bool cross_range_ok(const DevLevel &l, const double *x, const double *f, const double *out) {
    auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return l.pat && l.box_pair == 2 && (l.pat_w == 7 || l.pat_w == 5) && a16(x) && a16(f) && a16(out);
}
static void launch_jacobi_range(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *xin, const double *f,
                                double *xout, double omega, int64_t q_lo, int64_t q_hi) {
    if (q_hi <= q_lo) return;
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>((q_hi - q_lo + kCrossThreads - 1) / kCrossThreads, static_cast<int64_t>(l.box_grid))));
    if (l.pat_w == 7)
        launch_k(c, k_crosspair<M_JACOBI, 0, 7, true>, dim3(grid), dim3(kCrossThreads), l.pat_tb, s, static_cast<int>(l.n),
                 l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<7>(l), xin, f, xout, omega,
                 static_cast<const int *>(nullptr), Red{}, static_cast<int>(q_lo), static_cast<int>(q_hi));
    else
        launch_k(c, k_crosspair<M_JACOBI, 0, 5, true>, dim3(grid), dim3(kCrossThreads), l.pat_tb, s, static_cast<int>(l.n),
                 l.pat_id, l.pat_np, l.pat_table, l.box_rmask, main_pat<5>(l), xin, f, xout, omega,
                 static_cast<const int *>(nullptr), Red{}, static_cast<int>(q_lo), static_cast<int>(q_hi));
}

// TMA descriptor of an nx x ny x nz f64 grid at p with an (bx, by, 1) box,
// out-of-grid elements zero-filled; cached per context.
static CUtensorMap tmap3d(sb_ctx c, const double *p, int nx, int ny, int nz, int bx, int by, int bz = 1) {
    const auto key = std::make_tuple(static_cast<const void *>(p), nx, ny, nz, bx, by * 4096 + bz);
    auto it = c->tmaps.find(key);
    if (it != c->tmaps.end()) return it->second;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) throw sb::cuda_error("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    CUtensorMap m;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(nx), static_cast<cuuint64_t>(ny), static_cast<cuuint64_t>(nz)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(nx) * 8, static_cast<cuuint64_t>(nx) * ny * 8};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(by), static_cast<cuuint32_t>(bz)};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(p), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw sb::cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    c->tmaps.emplace(key, m);
    return m;
}

// two Jacobi sweeps xin -> out in one launch (k_cross_box2)
static void launch_box2(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *xin, const double *f,
                        double *out, double omega) {
    const BoxGeo &g = l.box_geo;
    const int TX = l.box_tx, TY = TX >= 16 ? 8 : 16, TZ = 8;
    const CUtensorMap mx = tmap3d(c, xin, g.nx, g.ny, g.nz, TX + 4, TY + 4, TZ + 4);
    const CUtensorMap mf = tmap3d(c, f, g.nx, g.ny, g.nz, TX + 4, TY + 2, TZ + 2);
    launch_k(c, box2_kernel(TX), dim3(l.tb_grid), dim3(kTbThreads), box2_smem(TX), s, mx, mf, g, l.tb_tab, out,
             omega, xin, f);
}

// two Jacobi sweeps xin -> out in one pass (k_cross_tb2)
static void launch_tb2(sb_ctx c, const DevLevel &l, cudaStream_t s, const double *xin, const double *f,
                       double *out, double omega) {
    if (l.tb == 2) return launch_box2(c, l, s, xin, f, out, omega);
    if (!kExperimental) throw sb::cuda_error("k_cross_tb2 is not built (SB_EXPERIMENTAL=0)");
    const TbGeo &g = l.tb_geo;
    const CUtensorMap mx = tmap3d(c, xin, g.nx, g.ny, g.nz, g.TX + 4, g.TY + 4);
    const CUtensorMap mf = tmap3d(c, f, g.nx, g.ny, g.nz, g.TX + 4, g.TY + 2);
    launch_k(c, tb_kernel(g.TX), dim3(l.tb_grid), dim3(kTbThreads), l.tb_smem, s, mx, mf, g, l.tb_tab, out, omega);
}

// How `count` consecutive Jacobi sweeps of level l are launched: fused pairs
// (k_cross_tb2) where the level has them, then a single sweep; last_single
// keeps the final launch a single sweep (it may carry the (r, z) reduction).
static std::vector<int> sweep_groups(const DevLevel &l, int count, bool last_single) {
    std::vector<int> g;
    if (!l.tb) {
        g.assign(static_cast<size_t>(std::max(count, 0)), 1);
        return g;
    }
    int left = count;
    while (left >= 2 && !(last_single && left == 2)) {
        g.push_back(2);
        left -= 2;
    }
    while (left-- > 0) g.push_back(1);
    return g;
}
static int sweep_launches(const DevLevel &l, int count, bool last_single) {
    return static_cast<int>(sweep_groups(l, count, last_single).size());
}

static void emit_coarse(sb_ctx c, cudaStream_t s, const double *f, double *x) {
    const int n = static_cast<int>(c->nc);
    if (c->coarse_exact)
        launch_k(c, k_coarse_lu_exact, dim3(1), dim3(32), sizeof(double) * n, s, n,
                 static_cast<const double *>(c->lu), static_cast<const int32_t *>(c->perm), f, x);
    else
        launch_k(c, k_coarse_gemv, dim3((n + 7) / 8), dim3(256), 0, s, n, static_cast<const double *>(c->inv), f,
                 x);
}

static void emit_tail(sb_ctx c, cudaStream_t s, const Cyc &cp, const double *f, double *X) {
    ++c->launch_count;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->tail_ctas, 1, 1);
    cfg.blockDim = dim3(kTailThreads, 1, 1);
    cfg.dynamicSmemBytes = static_cast<size_t>(c->tail_smem);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c->tail_ctas;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = c->pdl ? 2 : 1;
    CK(cudaLaunchKernelEx(&cfg, k_tail, static_cast<const TailDesc *>(c->tail), f, X, cp.omega, cp.pre, cp.post,
                          c->trace));
}

// Buffer the zero-guess first pre-sweep of level k writes (X = the level's
// output buffer; see emit_vcycle's buffer plan).
// (Each launch of a sweep group swaps the ping-pong pair; sweep_groups.)
static double *post_first_of(sb_ctx c, const Cyc &cp, int k, double *X) {
    const DevLevel &l = c->L[static_cast<size_t>(k)];
    return (cp.post >= 1) ? ((sweep_launches(l, cp.post - 1, k == 0) % 2 == 0) ? X : l.t) : X;
}
static double *zero_sweep_dest(sb_ctx c, const Cyc &cp, int k, double *X) {
    const DevLevel &l = c->L[static_cast<size_t>(k)];
    double *T = l.t;
    double *post_first = post_first_of(c, cp, k, X);
    double *pre_end = (cp.post >= 1) ? (post_first == X ? T : X) : X;
    return (sweep_launches(l, cp.pre - 1, false) % 2 == 0) ? pre_end : (pre_end == X ? T : X);
}

// Jacobi sweeps of level l in launch groups (1: one sweep, 2: k_cross_tb2),
// ping-ponging cur / other; the last single sweep carries `red` when given.
static void emit_sweeps(sb_ctx c, const DevLevel &l, cudaStream_t s, const std::vector<int> &groups, double *&cur,
                        double *&other, const double *f, double omega, const Red *red = nullptr,
                        bool *red_used = nullptr) {
    for (size_t i = 0; i < groups.size(); ++i) {
        if (groups[i] == 2) {
            launch_tb2(c, l, s, cur, f, other, omega);
        } else if (red && i + 1 == groups.size()) {
            launch_csr<M_JACOBI, 1>(c, l, s, cur, f, other, omega, nullptr, *red);
            if (red_used) *red_used = true;
        } else {
            launch_jacobi(c, l, s, cur, f, other, omega);
        }
        std::swap(cur, other);
    }
}

// One V-cycle at level k (cycle.hpp:53-75), result written to X. T is the
// level's ping-pong partner; the buffer plan makes the last post-sweep land
// in X without copies. From x = 0 the first sweep is x0 = 0 + w f / a_ii
// (k_jacobi_zero, or written by the parent's restriction when x0_ready);
// the prolongation + first post-sweep run fused. Levels
// from c->tail_from down run inside one cluster-resident kernel.
static void emit_vcycle(sb_ctx c, cudaStream_t s, const Cyc &cp, int k, const double *f, double *X,
                        bool zero, bool x0_ready = false) {
    const int L = static_cast<int>(c->L.size());
    if (k + 1 == L && !(zero && k == c->tail_from)) {
        emit_coarse(c, s, f, X);
        return;
    }
    if (zero && k == c->tail_from) {
        emit_tail(c, s, cp, f, X);
        return;
    }
    const DevLevel &l = c->L[static_cast<size_t>(k)];
    double *T = l.t;
    double *post_first = post_first_of(c, cp, k, X);
    double *cur = X, *other = T;
    if (zero) {
        double *pre_end = (cp.post >= 1) ? (post_first == X ? T : X) : X;
        if (cp.pre == 0) {
            CK(cudaMemsetAsync(pre_end, 0, sizeof(double) * static_cast<size_t>(l.n), s));
            cur = pre_end;
        } else {
            cur = zero_sweep_dest(c, cp, k, X);
            other = (cur == X) ? T : X;
            if (!x0_ready)
                launch_k(c, k_jacobi_zero, dim3(vec_grid(l.n)), dim3(kVecThreads), 0, s, l.n, f,
                         static_cast<const double *>(l.diag), cur, cp.omega);
            emit_sweeps(c, l, s, sweep_groups(l, cp.pre - 1, false), cur, other, f, cp.omega);
        }
    } else {
        emit_sweeps(c, l, s, sweep_groups(l, cp.pre, false), cur, other, f, cp.omega);
    }
    const DevLevel &lc = c->L[static_cast<size_t>(k) + 1];
    // the child's zero-guess sweep rides on the restriction (not for the
    // coarsest level or the cluster tail, which start from x = 0 themselves)
    const bool child_x0 = cp.pre >= 1 && k + 2 < L && k + 1 != c->tail_from;
    double *x0 = child_x0 ? zero_sweep_dest(c, cp, k + 1, lc.x) : nullptr;
    if (l.pat) {  // residual + restriction in one launch, no r vector
        launch_pat_rr(c, l, lc, s, cur, f, x0, cp.omega);
    } else {
        launch_csr<M_RESID, 0>(c, l, s, cur, f, c->rs, 0.0, nullptr, Red{});
        launch_k(c, k_restrict, dim3(vec_grid(lc.n)), dim3(kVecThreads), 0, s, lc.n,
                 static_cast<const int2 *>(l.mem), static_cast<const double *>(c->rs), lc.f,
                 static_cast<const double *>(lc.diag), x0, cp.omega);
    }
    emit_vcycle(c, s, cp, k + 1, lc.f, lc.x, true, child_x0);
    // On row-pair (7/5-point cross) levels the prolongation runs as its own
    // vector pass and every post-sweep as k_crosspair: measured faster at 256^3
    // than k_rowpat's fused prolongation + sweep; elsewhere the
    // prolongation rides on the first post-sweep's gathers.
    static const bool split_env = [] {
        const char *e = std::getenv("SB_PROLONG_SPLIT");
        return !(e && std::atoi(e) == 0);
    }();
    // aggregates = row pairs: the prolongation rides on k_crosspair's first
    // post-sweep (SB_PAIR_PC=0: the split form)
    static const bool pair_pc = [] {
        const char *e = std::getenv("SB_PAIR_PC");
        return !(e && std::atoi(e) == 0);
    }();
    auto a16p = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const bool fused_pair = pair_pc && l.pat && l.box_pair == 2 && l.pair_aggs && a16p(cur) && a16p(post_first) &&
                            a16p(f);
    const bool split = split_env && l.pat && l.box_pair == 2 && !fused_pair;
    if (cp.post >= 1 && cur != post_first && !split) {
        // x' = cur + P x_c folded into the first post-sweep's gathers
        launch_csr<M_JACOBI_PROLONG, 0>(c, l, s, cur, f, post_first, cp.omega, nullptr, Red{},
                                        Aux{l.diag, l.agg, lc.x});
        cur = post_first;
        other = (cur == X) ? T : X;
        // last kernel of the cycle at level 0: a single sweep + (z, r)
        emit_sweeps(c, l, s, sweep_groups(l, cp.post - 1, k == 0), cur, other, f, cp.omega,
                    k == 0 ? c->final_red : nullptr, &c->final_red_used);
    } else {
        double *pout = (sweep_launches(l, cp.post, k == 0) % 2 == 0) ? X : T;
        auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        if (l.n % 2 == 0 && a16(cur) && a16(pout) && a16(l.agg))
            launch_k(c, k_prolong2, dim3(vec_grid(l.n / 2)), dim3(kVecThreads), 0, s, l.n / 2,
                     reinterpret_cast<const int2 *>(l.agg), reinterpret_cast<const double2 *>(cur),
                     static_cast<const double *>(lc.x), reinterpret_cast<double2 *>(pout));
        else
            launch_k(c, k_prolong, dim3(vec_grid(l.n)), dim3(kVecThreads), 0, s, l.n,
                     static_cast<const int32_t *>(l.agg), static_cast<const double *>(cur),
                     static_cast<const double *>(lc.x), pout);
        cur = pout;
        other = (pout == X) ? T : X;
        // last kernel of the cycle at level 0: a single sweep + (z, r)
        emit_sweeps(c, l, s, sweep_groups(l, cp.post, k == 0), cur, other, f, cp.omega,
                    k == 0 ? c->final_red : nullptr, &c->final_red_used);
    }
}

// ---- graph construction helpers -------------------------------------------------

static cudaGraphConditionalHandle new_handle(cudaStream_t s) {
    if (tl_eager) return cudaGraphConditionalHandle{};
    cudaStreamCaptureStatus status;
    cudaGraph_t g;
    CK(cudaStreamGetCaptureInfo(s, &status, nullptr, &g, nullptr, nullptr));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
    return h;
}

static void add_cond(sb_ctx c, cudaStream_t s, int depth, cudaGraphConditionalHandle h,
                     cudaGraphConditionalNodeType type,
                     const std::function<void(cudaStream_t, int)> &body) {
    if (tl_eager) {  // host-side loop control: wait for the kernel that decided, read done
        auto done = [&]() {
            int d = 0;
            CK(cudaMemcpyAsync(&d, &c->st->done, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            return d != 0;
        };
        if (type == cudaGraphCondTypeWhile) {
            while (!done()) body(s, depth + 1);
        } else if (!done()) {
            body(s, depth + 1);
        }
        return;
    }
    cudaStreamCaptureStatus status;
    cudaGraph_t g;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &status, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams p{};

    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, deps, nd, &p));
    CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    cudaStream_t s2 = c->cap[depth];
    CK(cudaStreamBeginCaptureToGraph(s2, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeRelaxed));
    body(s2, depth + 1);
    cudaGraph_t out;
    CK(cudaStreamEndCapture(s2, &out));
}

static cudaGraph_t begin_capture(sb_ctx c) {
    if (tl_eager) return nullptr;
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    CK(cudaStreamBeginCaptureToGraph(c->stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    return g;
}

static cudaGraph_t end_capture(sb_ctx c, cudaGraph_t g) {
    if (tl_eager) return nullptr;
    cudaGraph_t out;
    CK(cudaStreamEndCapture(c->stream, &out));
    return g;
}

// X0 of level 0 (the first zero-guess sweep written by a Krylov update kernel)
static X0 level0_x0(sb_ctx c, double *x0, double omega) {
    const DevLevel &l0 = c->L[0];
    X0 z{static_cast<const double *>(l0.diag), x0, omega};
    if (x0 && l0.pat && l0.pat_np > 0) {
        z.pid = l0.pat_id;
        z.pdg = reinterpret_cast<const double *>(l0.pat_table) + static_cast<size_t>(l0.pat_np) * ((l0.pat_w + 1) & ~1);
        z.pry = z.pdg + l0.pat_np;
    }
    return z;
}

// PCG (krylov.hpp:65-119) as one graph: prologue IF (not converged at r0)
// { z = M r; p = z, rz; WHILE (!done) { Ap, pAp -> alpha; x, r, ||r|| ->
// tests; IF (!done) { z = M r; rz -> beta; p = z + beta p } } }; then the true
// residual. cp == nullptr: identity preconditioner (z = r).
static cudaGraph_t build_pcg(sb_ctx c, const Cyc *cp, const double *b, double *x) {
    // x += alpha p deferred into the p update (SB_DEFER_X=0: in the r update)
    static const bool defer_x = [] {
        const char *e = std::getenv("SB_DEFER_X");
        return !(e && std::atoi(e) == 0);
    }();
    const DevLevel &l0 = c->L[0];
    const int64_t n = l0.n;
    const int vb = vec_grid(n);
    double *r = c->kv[KR], *z = c->kv[KZ], *p = c->kv[KP], *Ap = c->kv[KAP];
    cudaStream_t s = c->stream;
    auto precond = [c, cp, n](cudaStream_t ss, const double *in, double *out, bool x0_ready) {
        if (cp) emit_vcycle(c, ss, *cp, 0, in, out, true, x0_ready);
        else CK(cudaMemcpyAsync(out, in, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToDevice, ss));
    };
    // the update kernel writes the V-cycle's first level-0 sweep when level 0
    // is an ordinary level with a pre-smoother
    const int L = static_cast<int>(c->L.size());
    double *x0 = (cp && cp->pre >= 1 && L >= 2 && c->tail_from != 0) ? zero_sweep_dest(c, *cp, 0, z) : nullptr;
    cudaGraph_t g = begin_capture(c);
    c->launch_count = 0;
    int mark = 0;
    auto plan = [&](int &field) {  // graph mode: kernels emitted since the last mark
        if (!tl_eager) field = c->launch_count - mark;
        mark = c->launch_count;
    };
    cudaGraphConditionalHandle h_pro = new_handle(s);
    launch_k(c, k_init, dim3(vb), dim3(kVecThreads), 0, s, n, b, x, r, make_red(c, EP_INIT_NORM, 1, nullptr, nullptr, conds({h_pro})));
    CK(cudaGetLastError());
    plan(c->plan.pre);
    add_cond(c, s, 0, h_pro, cudaGraphCondTypeIf, [&](cudaStream_t s1, int d1) {
        precond(s1, r, z, false);
        cudaGraphConditionalHandle h_loop = new_handle(s1);
        launch_k(c, k_copy_dot, dim3(vb), dim3(kVecThreads), 0, s1, n, z, p, nullptr, r,
                                              make_red(c, EP_PCG_RZ0, 1, nullptr, nullptr, conds({h_loop})), X0{});
        CK(cudaGetLastError());
        plan(c->plan.once);
        add_cond(c, s1, d1, h_loop, cudaGraphCondTypeWhile, [&](cudaStream_t s2, int d2) {
            launch_csr<M_SPMV, 1>(c, l0, s2, p, nullptr, Ap, 0.0, &c->st->done, make_red(c, EP_PCG_PAP, 1, p));
            cudaGraphConditionalHandle h_vc = new_handle(s2);
            if (defer_x)
                launch_k(c, k_pcg_update_r, dim3(vb), dim3(kVecThreads), 0, s2, n, r, static_cast<const double *>(Ap),
                         make_red(c, EP_PCG_RN, 1, nullptr, nullptr, conds({h_vc, h_loop})),
                         level0_x0(c, x0, cp ? cp->omega : 0.0));
            else
                launch_k(c, k_pcg_update, dim3(vb), dim3(kVecThreads), 0, s2,
                         n, x, r, p, Ap, make_red(c, EP_PCG_RN, 1, nullptr, nullptr, conds({h_vc, h_loop})),
                         level0_x0(c, x0, cp ? cp->omega : 0.0));
            CK(cudaGetLastError());
            plan(c->plan.per_it);
            add_cond(c, s2, d2, h_vc, cudaGraphCondTypeIf, [&](cudaStream_t s3, int) {
                const Red rz = make_red(c, EP_PCG_RZ, 1, r);
                c->final_red = &rz;  // (r, z) rides on the V-cycle's last sweep when it is a Jacobi sweep
                c->final_red_used = false;
                precond(s3, r, z, x0 != nullptr);
                c->final_red = nullptr;
                if (!c->final_red_used) {
                    launch_k(c, k_dot, dim3(vb), dim3(kVecThreads), 0, s3, n, r, z, nullptr, rz);
                    CK(cudaGetLastError());
                }
                if (defer_x)
                    launch_k(c, k_xpay_x, dim3(vb), dim3(kVecThreads), 0, s3, n, static_cast<const double *>(z), p, x,
                             c->st);
                else
                    launch_k(c, k_xpay, dim3(vb), dim3(kVecThreads), 0, s3, n, z, p, c->st);
                CK(cudaGetLastError());
                plan(c->plan.per_it_cond);
            });
        });
    });
    if (defer_x)  // the last iteration's x += alpha p
        launch_k(c, k_x_final, dim3(vb), dim3(kVecThreads), 0, s, n, x, static_cast<const double *>(p), c->st);
    // true residual ||b - A x|| (krylov.hpp:116)
    launch_csr<M_RESID, 1>(c, l0, s, x, b, c->rs, 0.0, nullptr, make_red(c, EP_STORE, 1));
    plan(c->plan.post);
    return end_capture(c, g);
}

// Flexible PBiCGStab (krylov.hpp:126-211).
static cudaGraph_t build_bicg(sb_ctx c, const Cyc *cp, const double *b, double *x) {
    const DevLevel &l0 = c->L[0];
    const int64_t n = l0.n;
    const int vb = vec_grid(n);
    double *r = c->kv[KR], *rbar = c->kv[KRBAR], *p = c->kv[KP], *pt = c->kv[KPT], *Apt = c->kv[KAPT],
           *sv = c->kv[KS], *stv = c->kv[KST], *Ast = c->kv[KAST];
    cudaStream_t s = c->stream;
    // the kernels producing p and s also write the first level-0 sweep of the
    // V-cycles that precondition them (X0)
    const int L = static_cast<int>(c->L.size());
    const bool fuse0 = cp && cp->pre >= 1 && L >= 2 && c->tail_from != 0;
    const X0 x0p = fuse0 ? level0_x0(c, zero_sweep_dest(c, *cp, 0, pt), cp->omega) : X0{};
    const X0 x0s = fuse0 ? level0_x0(c, zero_sweep_dest(c, *cp, 0, stv), cp->omega) : X0{};
    auto precond = [c, cp, n, fuse0](cudaStream_t ss, const double *in, double *out) {
        if (cp) emit_vcycle(c, ss, *cp, 0, in, out, true, fuse0);
        else CK(cudaMemcpyAsync(out, in, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToDevice, ss));
    };
    cudaGraph_t g = begin_capture(c);
    c->launch_count = 0;
    int mark = 0;
    auto plan = [&](int &field) {  // graph mode: kernels emitted since the last mark
        if (!tl_eager) field = c->launch_count - mark;
        mark = c->launch_count;
    };
    cudaGraphConditionalHandle h_pro = new_handle(s);
    launch_k(c, k_init, dim3(vb), dim3(kVecThreads), 0, s, n, b, x, r, make_red(c, EP_INIT_NORM, 1, nullptr, nullptr, conds({h_pro})));
    CK(cudaGetLastError());
    plan(c->plan.pre);
    add_cond(c, s, 0, h_pro, cudaGraphCondTypeIf, [&](cudaStream_t s1, int d1) {
        cudaGraphConditionalHandle h_loop = new_handle(s1);
        launch_k(c, k_copy_dot, dim3(vb), dim3(kVecThreads), 0, s1, n, r, rbar, p, r,
                                              make_red(c, EP_BI_RHO0, 1, nullptr, nullptr, conds({h_loop})), x0p);
        CK(cudaGetLastError());
        plan(c->plan.once);
        add_cond(c, s1, d1, h_loop, cudaGraphCondTypeWhile, [&](cudaStream_t s2, int d2) {
            // (the loop is only entered / re-entered with done == 0)
            precond(s2, p, pt);
            launch_csr<M_SPMV, 1>(c, l0, s2, pt, nullptr, Apt, 0.0, nullptr, make_red(c, EP_BI_DENOM, 1, rbar));
            cudaGraphConditionalHandle h_v2 = new_handle(s2);
            launch_k(c, k_bi_s, dim3(vb), dim3(kVecThreads), 0, s2, n, r, Apt, sv,
                                              make_red(c, EP_BI_SN, 1, nullptr, nullptr, conds({h_v2})), x0s);
            CK(cudaGetLastError());
            launch_k(c, k_bi_half, dim3(vb), dim3(kVecThreads), 0, s2, n, x, pt, c->st);
            CK(cudaGetLastError());
            plan(c->plan.per_it);
            add_cond(c, s2, d2, h_v2, cudaGraphCondTypeIf, [&](cudaStream_t s3, int) {
                precond(s3, sv, stv);
                launch_csr<M_SPMV, 2>(c, l0, s3, stv, nullptr, Ast, 0.0, nullptr,
                                      make_red(c, EP_BI_AS, 2, nullptr, sv));
                launch_k(c, k_bi_update, dim3(vb), dim3(kVecThreads), 0, s3, n, x, r, pt, stv, sv, Ast, rbar,
                                                       make_red(c, EP_BI_RN_RHO, 2));
                CK(cudaGetLastError());
                launch_k(c, k_bi_p, dim3(vb), dim3(kVecThreads), 0, s3, n, r, p, Apt, c->st, x0p);
                CK(cudaGetLastError());
                plan(c->plan.per_it_cond);
            });
            k_set_cond<<<1, 1, 0, s2>>>(c->st, conds({h_loop}));  // (eager: no handles, a no-op kernel)
            CK(cudaGetLastError());
            ++c->launch_count;
            if (!tl_eager) ++c->plan.per_it;  // k_set_cond runs every iteration
            mark = c->launch_count;
        });
    });
    launch_csr<M_RESID, 1>(c, l0, s, x, b, c->rs, 0.0, nullptr, make_red(c, EP_STORE, 1));
    plan(c->plan.post);
    return end_capture(c, g);
}

// Stationary AMG (cycle.hpp:91-130): WHILE (!done) { V-cycle(b, x); ||b - A x|| }.
static cudaGraph_t build_amg(sb_ctx c, const Cyc &cp, const double *b, double *x) {
    const DevLevel &l0 = c->L[0];
    const int64_t n = l0.n;
    const int vb = vec_grid(n);
    cudaStream_t s = c->stream;
    cudaGraph_t g = begin_capture(c);
    c->launch_count = 0;
    cudaGraphConditionalHandle h_loop = new_handle(s);
    launch_k(c, k_init, dim3(vb), dim3(kVecThreads), 0, s, n, b, x, nullptr,
                                      make_red(c, EP_INIT_NORM, 1, nullptr, nullptr, conds({h_loop})));
    CK(cudaGetLastError());
    if (!tl_eager) c->plan.pre = c->launch_count;
    add_cond(c, s, 0, h_loop, cudaGraphCondTypeWhile, [&](cudaStream_t s1, int) {
        const int m0 = c->launch_count;
        emit_vcycle(c, s1, cp, 0, b, x, false);
        launch_csr<M_RESID, 1>(c, l0, s1, x, b, c->rs, 0.0, nullptr,
                               make_red(c, EP_AMG_RN, 1, nullptr, nullptr, conds({h_loop})));
        if (!tl_eager) c->plan.per_it = c->launch_count - m0;
    });
    return end_capture(c, g);
}

// ---- context creation ----------------------------------------------------------

static void make_tiles(const HostCsr &A, std::vector<int32_t> &tiles, int &cap) {
    constexpr int64_t kCapMax = 4096;  // staged nnz per tile (49 KB per pipeline stage)
    tiles.assign(1, 0);
    cap = 0;
    int64_t r = 0;
    while (r < A.n) {
        int64_t r1 = r, nz = 0;
        while (r1 < A.n && r1 - r < kTileRows) {
            const int64_t len = A.rp[r1 + 1] - A.rp[r1];
            if (r1 > r && nz + len > kCapMax) break;
            nz += len;
            ++r1;
        }
        tiles.push_back(static_cast<int32_t>(r1));
        if (nz <= kCapMax) cap = std::max(cap, static_cast<int>(nz));
        r = r1;
    }
}

// Plane-marching sweep (sb_march.cuh) for a row-pattern level whose main
// pattern is a 27-point box: validate the box geometry of the main offsets,
// embed every pattern whose offsets are a subsequence of the main ones (values
// at the main slots, +0.0 elsewhere), upload the table. Opt-in (SB_MARCH=1);
// SB_MARCH_MIN: smallest level (rows) that gets it.
template <int G>
static bool march_geo_ok(const DevLevel &D, int &P, int &N) {
    constexpr int W = Geo<G>::W;
    if (D.main_len != W || static_cast<int>(D.main_o.size()) < W) return false;
    int kp = -1, kn = -1;  // slots (1, 0, 0) and (0, 1, 0)
    for (int k = 0; k < W; ++k) {
        if (Geo<G>::dz(k) == 1 && Geo<G>::dy(k) == 0 && Geo<G>::dx(k) == 0) kp = k;
        if (Geo<G>::dz(k) == 0 && Geo<G>::dy(k) == 1 && Geo<G>::dx(k) == 0) kn = k;
    }
    P = D.main_o[static_cast<size_t>(kp)];
    N = D.main_o[static_cast<size_t>(kn)];
    if (N < 32 || P % N != 0 || P / N < 2) return false;  // a tile row spans one line
    for (int k = 0; k < W; ++k)
        if (D.main_o[static_cast<size_t>(k)] != Geo<G>::dz(k) * P + Geo<G>::dy(k) * N + Geo<G>::dx(k)) return false;
    return true;
}

static void build_march(sb_ctx c, DevLevel &D, int np, int w, const double *val, const int32_t *off,
                        const uint8_t *len) {
    if (!kExperimental) return;
    const char *e = std::getenv("SB_MARCH");  // opt-in: measured slower than k_rowpat
    if (!e || std::atoi(e) == 0) return;
    const char *em = std::getenv("SB_MARCH_MIN");
    const int64_t nmin = em ? std::atoll(em) : 65536;
    if (D.n < nmin) return;
    int geo = -1, P = 0, N = 0;
    if (w == 28 && march_geo_ok<0>(D, P, N)) geo = 0;  // (7-point levels: the row-pattern kernel measured faster)
    if (geo < 0 || D.n / P < 3) return;
    const int W = D.main_len, WE = (W + 1) & ~1;
    const int wv = (w + 1) & ~1, wo = (w + 3) & ~3;
    const size_t mtb = march_table_bytes(np, W);
    std::vector<unsigned char> mt(mtb, 0);
    auto *ev = reinterpret_cast<double *>(mt.data());
    auto *emb = reinterpret_cast<uint8_t *>(ev + static_cast<size_t>(np) * WE);
    for (int q = 0; q < np; ++q) {
        int k = 0;
        for (int j = 0; j < W; ++j) {
            ev[q * WE + j] = 0.0;
            if (k < len[q] && off[q * wo + k] == D.main_o[static_cast<size_t>(j)]) ev[q * WE + j] = val[q * wv + k++];
        }
        emb[q] = (k == len[q]) ? 1 : 0;
    }
    auto *dt = dalloc<unsigned char>(c, static_cast<int64_t>(mtb));
    CK(cudaMemcpy(dt, mt.data(), mtb, cudaMemcpyHostToDevice));
    D.march_geo = geo;
    D.march_S = P;
    D.march_N = N;
    D.march_nqf = static_cast<int>(D.n / P);
    D.march_nxb = (N + 31) / 32;
    D.march_nyb = (P / N + kMarchLines - 1) / kMarchLines;
    const int nqb = (D.march_nqf - 2 + kMarchK - 1) / kMarchK;
    D.march_ntiles = D.march_nxb * D.march_nyb * nqb;
    D.march_tb = mtb;
    D.march_table = dt;
}

// Row-pattern format (§3.1): one byte per row when the level has <= 256
// distinct rows (offsets + value bits, CSR order) of length <= 32. Threads
// hash their rows, first occurrences become patterns, and every row is
// verified against its pattern's full key (a hash collision only disables the
// format). Returns false (nothing allocated) when the level does not qualify.
// Two-sweep temporal blocking (k_cross_tb2, sb_tblock.cuh): the level must be
// an nx x ny x nz grid in (iz*ny + iy)*nx + ix order whose row pattern is a
// function of the row's boundary class and whose absent slots are exactly the
// out-of-grid neighbours; checked for every row. SB_TB=0 disables it,
// SB_TB_MIN (rows, default 0) skips smaller levels.
static constexpr size_t kTbSmemMax = 112 * 1024;  // two CTAs per SM
// A structured 7-point level for the fused two-sweep kernels: an nx x ny x nz
// grid in (iz*ny + iy)*nx + ix order whose row pattern is a function of the
// row's boundary class and whose absent slots are exactly the out-of-grid
// neighbours (checked for every row). tab: per class the 7 values in CSR order
// (+0.0 where absent), a_ii, RN(1/a_ii).
static bool cross_classes(const DevLevel &D, const std::vector<uint8_t> &pid, const double *val, const int32_t *off,
                          const uint8_t *len, const double *dg, const double *ry, int64_t &nx, int64_t &ny,
                          int64_t &nz, std::vector<double> &tab) {
    const std::vector<int> &mo = D.main_o;
    if (D.main_len != 7 || mo.size() < 7) return false;
    const int64_t N = mo[5], P = mo[6], n = D.n;
    if (N < 2 || N % 2 != 0 || P % N != 0 || n % P != 0) return false;
    nx = N;
    ny = P / N;
    nz = n / P;
    if (ny < 2 || nz < 2 || nx > INT32_MAX / 2) return false;
    constexpr int wv = 8, wo = 8;  // SmemTab<7> row strides (doubles / int32)
    const int64_t want[7] = {-P, -N, -1, 0, 1, N, P};
    std::vector<int> cls_pat(kTbClasses, -1);
    auto cl = [](int64_t i, int64_t m) { return i == 0 ? 0 : (i == m - 1 ? 2 : 1); };
    for (int64_t m = 0; m < n; ++m) {
        const int64_t ix = m % nx, iy = (m / nx) % ny, iz = m / P;
        const int cx = cl(ix, nx), cy = cl(iy, ny), cz = cl(iz, nz), k = cx + 3 * cy + 9 * cz;
        const int q = pid[static_cast<size_t>(m)];
        if (cls_pat[k] < 0) {
            // the pattern's slots must be exactly the in-grid neighbours, in CSR order
            const bool present[7] = {iz > 0, iy > 0, ix > 0, true, ix < nx - 1, iy < ny - 1, iz < nz - 1};
            int j = 0;
            for (int sl = 0; sl < 7; ++sl) {
                if (!present[sl]) continue;
                if (j >= len[q] || off[q * wo + j] != want[sl]) return false;
                ++j;
            }
            if (j != len[q]) return false;
            cls_pat[k] = q;
        } else if (cls_pat[k] != q) {
            return false;
        }
    }
    tab.assign(kTbTab, 0.0);
    for (int k = 0; k < kTbClasses; ++k) {
        const int q = cls_pat[k];
        if (q < 0) continue;
        int j = 0;
        for (int sl = 0; sl < 7; ++sl)
            if (j < len[q] && off[q * wo + j] == want[sl]) tab[k * 9 + sl] = val[q * wv + j++];
        tab[k * 9 + 7] = dg[q];
        tab[k * 9 + 8] = ry[q];
    }
    return true;
}

// k_cross_box2 on the latency-bound mid levels (EXPERIMENTAL=1 and SB_BOX2=1;
// rows in [SB_BOX2_MIN, SB_BOX2_MAX] take it).
static void build_box2(sb_ctx c, DevLevel &D, const std::vector<uint8_t> &pid, const double *val,
                       const int32_t *off, const uint8_t *len, const double *dg, const double *ry) {
    if (!kExperimental) return;
    const char *e = std::getenv("SB_BOX2");  // opt-in: measured slower than two kernels
    if (!e || std::atoi(e) == 0) return;
    const char *emin = std::getenv("SB_BOX2_MIN"), *emax = std::getenv("SB_BOX2_MAX");
    const int64_t nmin = emin ? std::atoll(emin) : 0, nmax = emax ? std::atoll(emax) : (int64_t(1) << 20);
    if (D.n < nmin || D.n > nmax) return;
    int64_t nx = 0, ny = 0, nz = 0;
    std::vector<double> tab;
    if (!cross_classes(D, pid, val, off, len, dg, ry, nx, ny, nz, tab)) return;
    const int TX = nx >= 16 ? 16 : 8, TY = TX >= 16 ? 8 : 16, TZ = 8;
    if (nx < 8 || nx * 8 % 16 != 0) return;
    static const bool attr = [] {
        for (int tx : {16, 8})
            CK(cudaFuncSetAttribute(box2_kernel(tx), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(box2_smem(tx))));
        return true;
    }();
    (void)attr;
    BoxGeo g{};
    g.nx = static_cast<int>(nx);
    g.ny = static_cast<int>(ny);
    g.nz = static_cast<int>(nz);
    g.nbx = static_cast<int>((nx + TX - 1) / TX);
    g.nby = static_cast<int>((ny + TY - 1) / TY);
    g.nbz = static_cast<int>((nz + TZ - 1) / TZ);
    auto *dt = dalloc<double>(c, kTbTab);
    CK(cudaMemcpy(dt, tab.data(), sizeof(double) * kTbTab, cudaMemcpyHostToDevice));
    D.tb_tab = dt;
    D.box_geo = g;
    D.box_tx = TX;
    D.tb_grid = g.nbx * g.nby * g.nbz;
    D.tb = 2;
}

static void build_tb(sb_ctx c, DevLevel &D, const std::vector<uint8_t> &pid, int np, const double *val,
                     const int32_t *off, const uint8_t *len, const double *dg, const double *ry) {
    if (!kExperimental) return;
    const char *e = std::getenv("SB_TB");  // opt-in: measured slower
    if (!e || std::atoi(e) == 0) return;
    const char *em = std::getenv("SB_TB_MIN");
    if (em && D.n < std::atoll(em)) return;
    int64_t nx = 0, ny = 0, nz = 0;
    std::vector<double> tab;
    if (!cross_classes(D, pid, val, off, len, dg, ry, nx, ny, nz, tab)) return;
    (void)np;
    // tile: 64 x 16 columns (the whole x-line on narrow levels), <= kTbSmemMax of rings
    TbGeo g{};
    g.nx = static_cast<int>(nx);
    g.ny = static_cast<int>(ny);
    g.nz = static_cast<int>(nz);
    g.TX = 32;  // kernel instances: TX = 64, 32, 16, 8 with TY = 2 * kTbThreads / TX
    while (g.TX > nx && g.TX > 8) g.TX /= 2;
    if (g.TX > nx) return;
    g.TY = 2 * kTbThreads / g.TX;
    g.ntx = static_cast<int>((nx + g.TX - 1) / g.TX);
    g.nty = static_cast<int>((ny + g.TY - 1) / g.TY);
    static const bool attr = [] {
        for (int tx : {64, 32, 16, 8})
            CK(cudaFuncSetAttribute(tb_kernel(tx), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kTbSmemMax)));
        return true;
    }();
    (void)attr;
    const size_t smem = tb_smem_bytes(g.TX, g.TY);
    if (smem > kTbSmemMax) return;
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tb_kernel(g.TX), kTbThreads, smem));
    if (occ < 1) return;
    // z-chunks: minimise waves x steps per CTA (each CTA marches ZL + 4 planes)
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    const int64_t tiles = int64_t(g.ntx) * g.nty, res = int64_t(nsm) * occ;
    int best = 1;
    double best_cost = 1e300;
    for (int nch = 1; nch <= g.nz; ++nch) {
        const int zl = (g.nz + nch - 1) / nch;
        const int real = (g.nz + zl - 1) / zl;
        const double cost = static_cast<double>((tiles * real + res - 1) / res) * (zl + 4);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = real;
        }
    }
    g.ZL = (g.nz + best - 1) / best;
    auto *dt = dalloc<double>(c, kTbTab);
    CK(cudaMemcpy(dt, tab.data(), sizeof(double) * kTbTab, cudaMemcpyHostToDevice));
    D.tb_tab = dt;
    D.tb_geo = g;
    D.tb_smem = smem;
    D.tb_grid = static_cast<int>(tiles * ((g.nz + g.ZL - 1) / g.ZL));
    D.tb = 1;
}

static bool build_rpat(sb_ctx c, const HostCsr &A, DevLevel &D) {
    const char *pe = std::getenv("SB_RPAT");
    if ((pe && std::atoi(pe) == 0) || A.n == 0) return false;
    const int64_t n = A.n;
    auto row_hash = [&](int64_t i) {
        uint64_t h = 1469598103934665603ull ^ static_cast<uint64_t>(A.rp[i + 1] - A.rp[i]);
        for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
            uint64_t bits;
            std::memcpy(&bits, &A.v[e], 8);
            const uint64_t o = static_cast<uint64_t>(static_cast<int64_t>(A.ci[e]) - i);
            h = (h ^ o) * 1099511628211ull;
            h = (h ^ bits) * 1099511628211ull;
            h ^= h >> 29;
        }
        return h;
    };
    auto same_row = [&](int64_t a, int64_t b) {  // rows a and b have identical (offset, value) sequences
        const int64_t la = A.rp[a + 1] - A.rp[a];
        if (la != A.rp[b + 1] - A.rp[b]) return false;
        for (int64_t e = 0; e < la; ++e) {
            if (static_cast<int64_t>(A.ci[A.rp[a] + e]) - a != static_cast<int64_t>(A.ci[A.rp[b] + e]) - b) return false;
            if (std::memcmp(&A.v[A.rp[a] + e], &A.v[A.rp[b] + e], 8) != 0) return false;
        }
        return true;
    };
    // pass 1 (threads): per-row hash + each chunk's distinct hashes (first row of each)
    const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), n / 65536 + 1)));
    std::vector<uint64_t> hs(static_cast<size_t>(n));
    std::vector<std::vector<std::pair<uint64_t, int64_t>>> firsts(static_cast<size_t>(T));
    std::vector<int> too_many(static_cast<size_t>(T), 0), wide(static_cast<size_t>(T), 0);
    const int64_t per = (n + T - 1) / T;
    auto pass1 = [&](int t) {
        std::unordered_map<uint64_t, int64_t> seen;
        for (int64_t i = t * per; i < std::min<int64_t>(n, (t + 1) * per); ++i) {
            if (A.rp[i + 1] - A.rp[i] > 32) {
                wide[static_cast<size_t>(t)] = 1;
                return;
            }
            const uint64_t h = row_hash(i);
            hs[static_cast<size_t>(i)] = h;
            if (seen.emplace(h, i).second) {
                firsts[static_cast<size_t>(t)].push_back({h, i});
                if (seen.size() > 256) {
                    too_many[static_cast<size_t>(t)] = 1;
                    return;
                }
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back(pass1, t);
        for (auto &x : th) x.join();
    }
    for (int t = 0; t < T; ++t)
        if (too_many[static_cast<size_t>(t)] || wide[static_cast<size_t>(t)]) return false;
    std::unordered_map<uint64_t, int> ids;
    std::vector<int64_t> rep;  // representative row of each pattern
    for (int t = 0; t < T; ++t)
        for (auto &f : firsts[static_cast<size_t>(t)])
            if (ids.emplace(f.first, static_cast<int>(rep.size())).second) {
                rep.push_back(f.second);
                if (rep.size() > 256) return false;
            }
    // pass 2 (threads): pattern index per row, verified against the representative
    std::vector<uint8_t> pid(static_cast<size_t>(n));
    std::vector<int> bad(static_cast<size_t>(T), 0);
    auto pass2 = [&](int t) {
        for (int64_t i = t * per; i < std::min<int64_t>(n, (t + 1) * per); ++i) {
            const int q = ids.at(hs[static_cast<size_t>(i)]);
            if (!same_row(i, rep[static_cast<size_t>(q)])) {
                bad[static_cast<size_t>(t)] = 1;
                return;
            }
            pid[static_cast<size_t>(i)] = static_cast<uint8_t>(q);
        }
    };
    {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back(pass2, t);
        for (auto &x : th) x.join();
    }
    for (int t = 0; t < T; ++t)
        if (bad[static_cast<size_t>(t)]) return false;  // hash collision: use another format
    std::vector<uint64_t>().swap(hs);
    int wmax = 0;
    for (int64_t r : rep) wmax = std::max<int>(wmax, static_cast<int>(A.rp[r + 1] - A.rp[r]));
    const int w = wmax <= 5 ? 5 : wmax <= 7 ? 7 : wmax <= 8 ? 8 : wmax <= 16 ? 16 : wmax <= 28 ? 28 : 32;
    const int np = static_cast<int>(rep.size());
    const size_t tb = pat_table_bytes(np, w);
    std::vector<unsigned char> tab(tb, 0);
    const int wv = (w + 1) & ~1, wo = (w + 3) & ~3;  // 16-byte table rows (SmemTab)
    auto *val = reinterpret_cast<double *>(tab.data());
    auto *dg = val + static_cast<size_t>(np) * wv;
    auto *ry = dg + np;
    auto *off = reinterpret_cast<int32_t *>(ry + np);
    auto *len = reinterpret_cast<uint8_t *>(off + static_cast<size_t>(np) * wo);
    for (int q = 0; q < np; ++q) {
        const int64_t r = rep[static_cast<size_t>(q)];
        const int lq = static_cast<int>(A.rp[r + 1] - A.rp[r]);
        len[q] = static_cast<uint8_t>(lq);
        dg[q] = 0.0;
        for (int e = 0; e < w; ++e) {
            off[q * wo + e] = 0;  // padding: the row itself, value +0.0 (see k_rowpat)
            val[q * wv + e] = 0.0;
            if (e < lq) {
                off[q * wo + e] = static_cast<int32_t>(static_cast<int64_t>(A.ci[A.rp[r] + e]) - r);
                val[q * wv + e] = A.v[A.rp[r] + e];
                if (off[q * wo + e] == 0) dg[q] = val[q * wv + e];
            }
        }
        const double ad = std::fabs(dg[q]);
        ry[q] = (ad >= std::ldexp(1.0, -100) && ad <= std::ldexp(1.0, 100)) ? 1.0 / dg[q] : 0.0;
    }
    {  // the most frequent pattern goes to the kernels as a parameter (MainPat)
        std::vector<int64_t> cnt(static_cast<size_t>(np), 0);
        for (uint8_t q : pid) ++cnt[q];
        const int q = static_cast<int>(std::max_element(cnt.begin(), cnt.end()) - cnt.begin());
        D.main_p = q;
        D.main_len = len[q];
        D.main_d = dg[q];
        D.main_r = ry[q];
        D.main_v.assign(val + static_cast<size_t>(q) * wv, val + static_cast<size_t>(q) * wv + w);
        D.main_o.assign(off + static_cast<size_t>(q) * wo, off + static_cast<size_t>(q) * wo + w);
    }
    build_march(c, D, np, w, val, off, len);
    {  // row-pair kernels: main pattern a 27-point box (k_boxpair) or a 7/5-point
       // cross (k_crosspair) with even strides, n even
        const char *bp = std::getenv("SB_BOXPAIR");
        int P = 0, N = 0, kind = 0;
        const std::vector<int> &mo = D.main_o;
        if (!(bp && std::atoi(bp) == 0) && A.n % 2 == 0 && A.n >= 2) {
            if (w == 28 && march_geo_ok<0>(D, P, N) && P % 2 == 0 && N % 2 == 0) kind = 1;
            if (w == 7 && D.main_len == 7 && mo[0] == -mo[6] && mo[1] == -mo[5] && mo[2] == -1 && mo[3] == 0 &&
                mo[4] == 1 && mo[5] > 1 && mo[6] > mo[5] && mo[5] % 2 == 0 && mo[6] % 2 == 0)
                kind = 2;
            // 5-point 2D cross: faster on large levels (C1 L0 5.3 vs 5.7 us) but slower
            // on 2D coarse levels (V-cycle 0.364 vs 0.343 ms with every level), so
            // only levels >= 2^19 rows (SB_CROSS5=1: every level, =0: none)
            const char *c5 = std::getenv("SB_CROSS5");
            const bool c5_on = c5 ? std::atoi(c5) != 0 : A.n >= (int64_t(1) << 19);
            if (c5_on && w == 5 && D.main_len == 5 && mo[0] == -mo[4] && mo[1] == -1 &&
                mo[2] == 0 && mo[3] == 1 && mo[4] > 1 && mo[4] % 2 == 0)
                kind = 2;
        }
        if (kind) {
            // restriction masks: pattern q = the main pattern with slots removed
            // (same offsets in order, same value bits where present), else 0
            const int wv = (w + 1) & ~1, wo = (w + 3) & ~3, W = D.main_len;
            std::vector<uint32_t> rm(static_cast<size_t>(np), 0u);
            for (int q = 0; q < np; ++q) {
                uint32_t m = 0u;
                int k = 0;
                for (int j = 0; j < W; ++j)
                    if (k < len[q] && off[q * wo + k] == mo[static_cast<size_t>(j)]) {
                        if (std::memcmp(&val[q * wv + k], &D.main_v[static_cast<size_t>(j)], 8) != 0) break;
                        m |= 1u << j;
                        ++k;
                    }
                rm[static_cast<size_t>(q)] = (k == len[q]) ? m : 0u;
            }
            auto *dm = dalloc<uint32_t>(c, np);
            CK(cudaMemcpy(dm, rm.data(), sizeof(uint32_t) * rm.size(), cudaMemcpyHostToDevice));
            D.box_rmask = dm;
            D.box_pair = kind;
        }
    }
    if (D.box_pair == 2 && w == 7) {
        build_tb(c, D, pid, np, val, off, len, dg, ry);
        if (!D.tb) build_box2(c, D, pid, val, off, len, dg, ry);
    }
    auto *dp = dalloc<uint8_t>(c, A.n + 16);
    CK(cudaMemcpy(dp, pid.data(), pid.size(), cudaMemcpyHostToDevice));
    auto *dt = dalloc<unsigned char>(c, static_cast<int64_t>(tb));
    CK(cudaMemcpy(dt, tab.data(), tb, cudaMemcpyHostToDevice));
    D.pat = 1;
    D.pat_np = np;
    D.pat_w = w;
    D.pat_tb = tb;
    D.pat_id = dp;
    D.pat_table = dt;
    return true;
}

// Matrix part of a level: diagonal, then the first format that applies: row
// patterns (RPAT), grouped sliced-ELL (SELL-G), CSR tiles. Columns need not be
// sorted (partitioned levels number ghosts after own rows).
static void upload_matrix(sb_ctx c, const HostCsr &A, DevLevel &D) {
    D.n = A.n;
    D.nnz = A.nnz();
    // diagonal + first bad row (smoother.hpp:55-70)
    std::vector<double> diag(static_cast<size_t>(A.n), 0.0);
    D.bad_diag = -1;
    for (int64_t i = 0; i < A.n; ++i) {
        int64_t pos = -1;
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k)
            if (A.ci[k] == i) pos = k;
        if (pos < 0 || A.v[pos] == 0.0) {
            if (D.bad_diag < 0) D.bad_diag = i;
        } else {
            diag[i] = A.v[pos];
        }
    }
    D.diag = dalloc<double>(c, A.n);
    CK(cudaMemcpy(D.diag, diag.data(), sizeof(double) * diag.size(), cudaMemcpyHostToDevice));
    if (A.n > INT32_MAX - 1024) throw invalid_argument("sb_create: level too large for int32 row indices");
    if (build_rpat(c, A, D)) return;  // 1 B/row: no other copy of the matrix on the device
    if (A.nnz() > INT32_MAX - 16)
        throw invalid_argument("sb_create: level too large for int32 device offsets (and not row-pattern)");
    std::vector<int32_t> rp32(static_cast<size_t>(A.n) + 1);
    for (int64_t i = 0; i <= A.n; ++i) rp32[i] = static_cast<int32_t>(A.rp[i]);
    D.rp = dalloc<int32_t>(c, A.n + 1 + 8);  // + slack for 16-byte TMA windows
    D.ci = dalloc<int32_t>(c, A.nnz() + 8);
    D.v = dalloc<double>(c, A.nnz() + 2);
    CK(cudaMemcpy(D.rp, rp32.data(), sizeof(int32_t) * rp32.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(D.ci, A.ci.data(), sizeof(int32_t) * A.ci.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(D.v, A.v.data(), sizeof(double) * A.v.size(), cudaMemcpyHostToDevice));
    std::vector<int32_t> tiles;
    make_tiles(A, tiles, D.cap);
    D.ntiles = static_cast<int>(tiles.size()) - 1;
    D.tiles = dalloc<int32_t>(c, static_cast<int64_t>(tiles.size()));
    CK(cudaMemcpy(D.tiles, tiles.data(), sizeof(int32_t) * tiles.size(), cudaMemcpyHostToDevice));
    // lossless streamed format: dictionary values / int16 column deltas
    const char *cz = std::getenv("SB_COMPRESS");
    const bool compress = !cz || std::atoi(cz) != 0;
    D.sv = D.v;
    D.sc = D.ci;
    if (compress && A.nnz() > 0) {
        std::map<uint64_t, int> ids;
        std::vector<double> dict;
        bool ok = true;
        for (int64_t k = 0; k < A.nnz() && ok; ++k) {
            uint64_t bits;
            std::memcpy(&bits, &A.v[k], 8);
            if (ids.find(bits) == ids.end()) {
                if (dict.size() == 256) ok = false;
                else {
                    ids[bits] = static_cast<int>(dict.size());
                    dict.push_back(A.v[k]);
                }
            }
        }
        if (ok) {
            std::vector<uint8_t> vi(static_cast<size_t>(A.nnz()));
            for (int64_t k = 0; k < A.nnz(); ++k) {
                uint64_t bits;
                std::memcpy(&bits, &A.v[k], 8);
                vi[k] = static_cast<uint8_t>(ids[bits]);
            }
            auto *dvi = dalloc<uint8_t>(c, A.nnz() + 32);
            CK(cudaMemcpy(dvi, vi.data(), vi.size(), cudaMemcpyHostToDevice));
            D.dict = dalloc<double>(c, 256);
            CK(cudaMemcpy(D.dict, dict.data(), sizeof(double) * dict.size(), cudaMemcpyHostToDevice));
            D.sv = dvi;
            D.vf = 1;
            D.ndict = static_cast<int>(dict.size());
        }
        bool fits = true;
        for (int64_t i = 0; i < A.n && fits; ++i)
            for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                const int64_t dlt = static_cast<int64_t>(A.ci[k]) - i;
                if (dlt < -32768 || dlt > 32767) {
                    fits = false;
                    break;
                }
            }
        if (fits) {
            std::vector<int16_t> cd(static_cast<size_t>(A.nnz()));
            for (int64_t i = 0; i < A.n; ++i)
                for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) cd[k] = static_cast<int16_t>(A.ci[k] - i);
            auto *dcd = dalloc<int16_t>(c, A.nnz() + 16);
            CK(cudaMemcpy(dcd, cd.data(), sizeof(int16_t) * cd.size(), cudaMemcpyHostToDevice));
            D.sc = dcd;
            D.cf = 1;
        }
    }
    D.smem = kStages * stage_bytes_of(D.cap, D.vf, D.cf);  // pipeline stages
    // grouped sliced-ELL conversion (SB_SELL=0 keeps the CSR pipeline)
    const char *se = std::getenv("SB_SELL");
    if ((!se || std::atoi(se) != 0) && A.n > 0) {
        const int64_t H = kTileRows;
        const int64_t nt = (A.n + H - 1) / H;
        std::vector<int> wt(static_cast<size_t>(nt), 0);
        int wmax = 0;
        for (int64_t t = 0; t < nt; ++t) {
            int w = 0;
            for (int64_t r = t * H; r < std::min<int64_t>(A.n, (t + 1) * H); ++r)
                w = std::max<int>(w, static_cast<int>(A.rp[r + 1] - A.rp[r]));
            wt[static_cast<size_t>(t)] = w;
            wmax = std::max(wmax, w);
        }
        // group size: 4 (fewest instructions) unless 2 saves > 5% of the slots
        int64_t s2 = 0, s4 = 0;
        for (int w : wt) {
            s2 += (w + 1) / 2 * 2;
            s4 += (w + 3) / 4 * 4;
        }
        const int gs = (s4 * 100 <= s2 * 105) ? 4 : 2;
        const int ngmax = (wmax + gs - 1) / gs;
        const int64_t slots = (gs == 4 ? s4 : s2) * H;
        const size_t stage = sg_stage_bytes(ngmax, gs, static_cast<int>(H), D.vf, D.cf);
        const bool ok = wmax <= 255 && slots <= 3 * A.nnz() / 2 + H && kSgStages * stage <= 200 * 1024;
        if (ok) {
            const int VB = D.vf ? 1 : 8, CB = D.cf ? 2 : 4;
            std::vector<int64_t> off(static_cast<size_t>(nt) + 1, 0);
            for (int64_t t = 0; t < nt; ++t) {
                const int ng = (wt[static_cast<size_t>(t)] + gs - 1) / gs;
                off[static_cast<size_t>(t) + 1] = off[static_cast<size_t>(t)] +
                    static_cast<int64_t>(sg_block_bytes(ng, gs, static_cast<int>(H), D.vf, D.cf));
            }
            std::vector<unsigned char> blk(static_cast<size_t>(off[static_cast<size_t>(nt)]), 0);
            std::map<uint64_t, int> ids;
            std::vector<double> dict;
            if (D.vf) {  // same dictionary order as the CSR-stream arrays
                dict.resize(static_cast<size_t>(D.ndict));
                CK(cudaMemcpy(dict.data(), D.dict, sizeof(double) * dict.size(), cudaMemcpyDeviceToHost));
                for (int q = 0; q < D.ndict; ++q) {
                    uint64_t bits;
                    std::memcpy(&bits, &dict[static_cast<size_t>(q)], 8);
                    ids[bits] = q;
                }
            }
            for (int64_t t = 0; t < nt; ++t) {
                const int ng = (wt[static_cast<size_t>(t)] + gs - 1) / gs;
                unsigned char *b = blk.data() + off[static_cast<size_t>(t)];
                int lmin = 1 << 30;
                for (int64_t r = t * H; r < std::min<int64_t>(A.n, (t + 1) * H); ++r)
                    lmin = std::min<int>(lmin, static_cast<int>(A.rp[r + 1] - A.rp[r]));
                const int32_t hd[4] = {ng, std::min(ng, lmin / gs), 0, 0};
                std::memcpy(b, hd, sizeof hd);
                unsigned char *bv = b + kSgHdr;
                unsigned char *bc = bv + static_cast<size_t>(ng) * H * gs * VB;
                unsigned char *bm = bc + static_cast<size_t>(ng) * H * gs * CB;
                for (int64_t r = t * H; r < std::min<int64_t>(A.n, (t + 1) * H); ++r) {
                    const int64_t lr = r - t * H;
                    const int64_t len = A.rp[r + 1] - A.rp[r];
                    int di = 0;  // diagonal: dictionary index (vf) or slot (a missing one is rejected before a sweep)
                    for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k)
                        if (A.ci[k] == r) {
                            if (D.vf) {
                                uint64_t bits;
                                std::memcpy(&bits, &A.v[k], 8);
                                di = ids[bits];
                            } else {
                                di = static_cast<int>(k - A.rp[r]);
                            }
                        }
                    const uint16_t m = static_cast<uint16_t>(len | (di << 8));
                    std::memcpy(bm + 2 * lr, &m, 2);
                    for (int64_t e = 0; e < static_cast<int64_t>(ng) * gs; ++e) {
                        const size_t pos = static_cast<size_t>((e / gs) * H + lr) * gs + static_cast<size_t>(e % gs);
                        int64_t col = r;  // padding: column = row, value index 0 / 0.0 (predicated out)
                        double val = 0.0;
                        int vi = 0;
                        if (e < len) {
                            const int64_t k = A.rp[r] + e;
                            col = A.ci[k];
                            val = A.v[k];
                            if (D.vf) {
                                uint64_t bits;
                                std::memcpy(&bits, &A.v[k], 8);
                                vi = ids[bits];
                            }
                        }
                        if (D.vf) bv[pos] = static_cast<uint8_t>(vi);
                        else std::memcpy(bv + pos * 8, &val, 8);
                        if (D.cf) {
                            const int16_t dl = static_cast<int16_t>(col - r);
                            std::memcpy(bc + pos * 2, &dl, 2);
                        } else {
                            const int32_t cc = static_cast<int32_t>(col);
                            std::memcpy(bc + pos * 4, &cc, 4);
                        }
                    }
                }
            }
            D.soff = dalloc<int64_t>(c, nt + 1);
            CK(cudaMemcpy(D.soff, off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice));
            auto *p = dalloc<unsigned char>(c, static_cast<int64_t>(blk.size()) + 16);
            CK(cudaMemcpy(p, blk.data(), blk.size(), cudaMemcpyHostToDevice));
            D.sell_blk = p;
            if (D.vf) {  // Markstein reciprocals RN(1/d); 0 where |d| leaves [2^-100, 2^100]
                std::vector<double> rd(dict.size(), 0.0);
                for (size_t q = 0; q < dict.size(); ++q) {
                    const double d = std::fabs(dict[q]);
                    if (d >= std::ldexp(1.0, -100) && d <= std::ldexp(1.0, 100)) rd[q] = 1.0 / dict[q];
                }
                D.rdict = dalloc<double>(c, 256);
                CK(cudaMemcpy(D.rdict, rd.data(), sizeof(double) * rd.size(), cudaMemcpyHostToDevice));
            }
            D.sell = 1;
            D.sell_tiles = static_cast<int>(nt);
            D.sell_ngmax = ngmax;
            D.sell_gs = gs;
            D.sell_slots = slots;
            D.sell_smem = kSgStages * stage;
        }
    }
}

static void upload_level(sb_ctx c, const HostLevel &H, DevLevel &D, bool coarsest, int64_t n0) {
    const HostCsr &A = H.A;
    // hybrid mode (paper's MI placement): matrix storage of levels >= host_from in host memory
    c->alloc_host = (&D - c->L.data()) >= c->host_from;
    upload_matrix(c, A, D);
    c->alloc_host = false;
    if (!coarsest) {
        D.nc = H.n_coarse;
        D.agg = dalloc<int32_t>(c, A.n);
        CK(cudaMemcpy(D.agg, H.agg.data(), sizeof(int32_t) * H.agg.size(), cudaMemcpyHostToDevice));
        std::vector<int2> mem(static_cast<size_t>(D.nc), make_int2(-1, -1));
        for (int64_t i = 0; i < A.n; ++i) {
            int2 &m = mem[static_cast<size_t>(H.agg[i])];
            if (m.x < 0) m.x = static_cast<int>(i);
            else m.y = static_cast<int>(i);
        }
        D.mem = dalloc<int2>(c, D.nc);
        CK(cudaMemcpy(D.mem, mem.data(), sizeof(int2) * mem.size(), cudaMemcpyHostToDevice));
        // every aggregate the row pair (2c, 2c + 1) (node-HEM on a grid level)
        D.pair_aggs = A.n % 2 == 0 && D.nc == A.n / 2;
        for (int64_t q = 0; D.pair_aggs && q < D.nc; ++q)
            D.pair_aggs = mem[static_cast<size_t>(q)].x == 2 * q && mem[static_cast<size_t>(q)].y == 2 * q + 1;
    }
    D.t = dalloc<double>(c, A.n);
    if (A.n != n0 || &D != &c->L[0]) {  // level 0 uses the caller's / Krylov vectors
        D.x = dalloc<double>(c, A.n);
        D.f = dalloc<double>(c, A.n);
    }
}

template <int MODE, int NV, int VF, int CF> static void set_sg_attr(int b) {
    CK(cudaFuncSetAttribute(k_sellg<MODE, NV, VF, CF, 4, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(k_sellg<MODE, NV, VF, CF, 2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    if constexpr (VF == 1 && CF == 1) {
        CK(cudaFuncSetAttribute(k_sellg<MODE, NV, 1, 1, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_sellg<MODE, NV, 1, 1, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_sellg<MODE, NV, 1, 1, 4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_sellg<MODE, NV, 1, 1, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_sellg<MODE, NV, 1, 1, 4, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_sellg<MODE, NV, 1, 1, 4, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_sellg<MODE, NV, 1, 1, 4, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    }
}

template <int MODE, int NV> static void set_smem_attr(size_t smem) {
    if (smem <= 48 * 1024) return;
    const int b = static_cast<int>(smem);
    if constexpr (MODE == M_JACOBI || MODE == M_SPMV || MODE == M_RESID) {
        CK(cudaFuncSetAttribute(k_boxpair<MODE, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_crosspair<MODE, NV, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_crosspair<MODE, NV, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        if constexpr (kExperimental) {
            if constexpr (MODE == M_RESID && NV == 0)
                CK(cudaFuncSetAttribute(k_cross_rr<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
            CK(cudaFuncSetAttribute(k_march<MODE, NV, 0, 28, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
            CK(cudaFuncSetAttribute(k_march<MODE, NV, 0, 28, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        }
    }
    CK(cudaFuncSetAttribute(k_rowpat<MODE, NV, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(k_rowpat<MODE, NV, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(k_rowpat<MODE, NV, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(k_rowpat<MODE, NV, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(k_rowpat<MODE, NV, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    if constexpr (MODE == M_RESID && NV == 0) {
        CK(cudaFuncSetAttribute(k_pat_resid_restrict<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_pat_resid_restrict<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_pat_resid_restrict<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_pat_resid_restrict<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_pat_resid_restrict<28>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        CK(cudaFuncSetAttribute(k_pat_resid_restrict<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    }
    CK(cudaFuncSetAttribute(k_rowpat<MODE, NV, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    set_sg_attr<MODE, NV, 0, 0>(b);
    set_sg_attr<MODE, NV, 1, 0>(b);
    set_sg_attr<MODE, NV, 0, 1>(b);
    set_sg_attr<MODE, NV, 1, 1>(b);
    CK(cudaFuncSetAttribute(k_csr_tile<MODE, NV, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(k_csr_tile<MODE, NV, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(k_csr_tile<MODE, NV, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(k_csr_tile<MODE, NV, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
}

static Cyc check_cycle(sb_ctx c, const sb_cycle *cp, const char *who) {
    Cyc y;
    if (!cp) return y;
    if (cp->smoother != SB_SMOOTHER_JACOBI)
        throw invalid_argument(std::string(who) +
                               ": only the weighted Jacobi smoother runs on the device (Gauss-Seidel "
                               "is inherently sequential and is not emulated)");
    if (!(cp->omega > 0.0) || cp->omega > 1.0)
        throw invalid_argument("SmootherKind: Jacobi weight " + std::to_string(cp->omega) +
                               " outside (0, 1]");
    if (cp->pre_sweeps < 0 || cp->post_sweeps < 0)
        throw invalid_argument("smooth: negative sweep count");
    y.pre = cp->pre_sweeps;
    y.post = cp->post_sweeps;
    y.omega = cp->omega;
    if (y.pre + y.post > 0)
        for (size_t k = 0; k + 1 < c->L.size(); ++k)
            if (c->L[k].bad_diag >= 0)
                throw invalid_argument("smooth: zero diagonal entry in row " +
                                       std::to_string(c->L[k].bad_diag));
    if (c->nc <= 0) throw invalid_argument(std::string(who) + ": hierarchy has no coarse factorization");
    return y;
}

// Chooses the cluster-resident tail: starting from the coarsest level, adds
// finer levels while each CTA's block of every tail level (CSR slice, diag,
// aggregates, members, 4 vectors) plus its rows of the coarse inverse fit in
// shared memory. SB_TAIL_ROWS caps the finest tail level (0 disables; default
// 1<<20). Disabled in the bit-exact coarse mode.
static void setup_tail(sb_ctx c, const Hier &H) {
    const int L = static_cast<int>(c->L.size());
    c->tail_from = 1 << 30;
    const char *env = std::getenv("SB_TAIL_ROWS");
    const long long tail_rows = env ? std::atoll(env) : 8192;  // measured: C2 tail from 8192 rows beats 16384 (tools/level_costs.py)
    if (tail_rows <= 0 || c->nc <= 0 || c->coarse_exact || L < 2) return;
    CK(cudaFuncSetAttribute(k_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int dev_smem = 0;
    CK(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    const int budget = dev_smem - static_cast<int>(sizeof(TailDesc)) - 1024;
    int ctas = 0;
    const char *ce = std::getenv("SB_TAIL_CTAS");
    for (int want : {16, 8, 4}) {
        if (ce && std::atoi(ce) != want) continue;
        CK(cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(want, 1, 1);
        cfg.blockDim = dim3(kTailThreads, 1, 1);
        cfg.dynamicSmemBytes = budget;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = want;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, k_tail, &cfg) == cudaSuccess && nclusters > 0) {
            ctas = want;
            break;
        }
        cudaGetLastError();
    }
    if (ctas == 0) return;
    auto a16 = [](int64_t x) { return (x + 15) & ~int64_t(15); };
    const int nc = static_cast<int>(c->nc);
    const int rows_c = (nc + ctas - 1) / ctas;
    auto rows_per_of = [&](int k) {
        return k == L - 1 ? rows_c : static_cast<int>((H.levels[static_cast<size_t>(k)].A.n + ctas - 1) / ctas);
    };
    // per level: rows per CTA, max local nnz, per-CTA ghost lists, value dictionary (<= 256 distinct)
    struct LevInfo {
        int rows_per = 0, nnz_cap = 0, gh_cap = 0, vf = 0;
        std::vector<std::vector<int64_t>> ghosts;  // per CTA: sorted remote columns
        std::vector<double> dict;
        std::map<uint64_t, int> ids;
    };
    std::vector<LevInfo> info(static_cast<size_t>(L));
    auto level_bytes = [&](int k) -> int64_t {  // image + vectors of a non-coarsest tail level, per CTA
        LevInfo &li = info[static_cast<size_t>(k)];
        const HostCsr &A = H.levels[static_cast<size_t>(k)].A;
        li.rows_per = rows_per_of(k);
        li.nnz_cap = li.gh_cap = 0;
        li.ghosts.assign(static_cast<size_t>(ctas), {});
        for (int r = 0; r < ctas; ++r) {
            const int64_t a = std::min<int64_t>(A.n, static_cast<int64_t>(r) * li.rows_per);
            const int64_t b = std::min<int64_t>(A.n, static_cast<int64_t>(r + 1) * li.rows_per);
            li.nnz_cap = std::max<int>(li.nnz_cap, static_cast<int>(A.rp[b] - A.rp[a]));
            std::vector<int64_t> &g = li.ghosts[static_cast<size_t>(r)];
            for (int64_t e = A.rp[a]; e < A.rp[b]; ++e)
                if (A.ci[e] < a || A.ci[e] >= b) g.push_back(A.ci[e]);
            std::sort(g.begin(), g.end());
            g.erase(std::unique(g.begin(), g.end()), g.end());
            li.gh_cap = std::max<int>(li.gh_cap, static_cast<int>(g.size()));
        }
        li.dict.clear();
        li.ids.clear();
        li.vf = 1;
        for (int64_t e = 0; e < A.nnz() && li.vf; ++e) {
            uint64_t bits;
            std::memcpy(&bits, &A.v[e], 8);
            if (li.ids.find(bits) == li.ids.end()) {
                if (li.dict.size() == 256) li.vf = 0;
                else {
                    li.ids[bits] = static_cast<int>(li.dict.size());
                    li.dict.push_back(A.v[e]);
                }
            }
        }
        if (li.rows_per + li.gh_cap > 65535) return INT64_MAX / 4;
        const int rpc = rows_per_of(k + 1);
        const int vb = li.vf ? 1 : 8;
        return a16(4 * (li.rows_per + 1)) + a16(2 * li.nnz_cap) + a16(vb * li.nnz_cap) + a16(vb * li.rows_per) +
               a16(4 * li.gh_cap) + a16(4 * li.rows_per) + a16(8 * rpc) +
               (li.vf ? 2 * a16(8 * static_cast<int64_t>(li.dict.size())) : 0) +
               2 * a16(8 * (li.rows_per + li.gh_cap)) + 2 * a16(8 * li.rows_per);
    };
    int64_t total = a16(4 * kTailMaxLevels) + a16(8 * static_cast<int64_t>(rows_c) * nc) + a16(8 * nc) +
                    2 * a16(8 * rows_c);
    int k0 = L - 1;
    while (k0 > c->tail_min) {
        const int k = k0 - 1;
        if (c->L[static_cast<size_t>(k)].n > tail_rows || L - k > kTailMaxLevels) break;
        if ((H.levels[static_cast<size_t>(k)].A.n + ctas - 1) / ctas > 32768) break;
        {  // the tail sums a row per thread: levels with long (hub) rows stay on
           // the kernels, whose CSR tiles give such rows a whole warp
            const HostCsr &A = H.levels[static_cast<size_t>(k)].A;
            int64_t wmax = 0;
            for (int64_t i = 0; i < A.n; ++i) wmax = std::max<int64_t>(wmax, A.rp[i + 1] - A.rp[i]);
            if (wmax > kLongRow) break;
        }
        const int64_t add = level_bytes(k);
        if (total + add > budget) break;
        total += add;
        k0 = k;
    }
    if (k0 >= L - 1) return;  // nothing above the coarsest fits
    for (int k = k0; k + 1 < L; ++k) level_bytes(k);  // (re-)fill info for the chosen levels
    TailDesc d;
    std::memset(&d, 0, sizeof(d));
    d.nlev = L - k0;
    d.ncoarse = nc;
    d.rows_c = rows_c;
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        const int64_t o = off;
        off += a16(bytes);
        return static_cast<int>(o);
    };
    take(4 * kTailMaxLevels);  // per-level ghost counts of this CTA
    for (int q = 0; q + 1 < d.nlev; ++q) {
        const int k = k0 + q;
        const LevInfo &li = info[static_cast<size_t>(k)];
        TailLevel &t = d.L[q];
        const int vb = li.vf ? 1 : 8;
        t.n = static_cast<int>(H.levels[static_cast<size_t>(k)].A.n);
        t.rows_per = li.rows_per;
        t.gh_cap = li.gh_cap;
        t.vf = li.vf;
        t.ndict = static_cast<int>(li.dict.size());
        t.o_rp = take(4 * (li.rows_per + 1));
        t.o_col = take(2 * li.nnz_cap);
        t.o_val = take(vb * li.nnz_cap);
        t.o_dix = take(vb * li.rows_per);
        t.o_gh = take(4 * li.gh_cap);
        t.o_agg = take(4 * li.rows_per);
        t.o_mem = take(8 * rows_per_of(k + 1));
        t.o_dict = li.vf ? take(8 * t.ndict) : 0;
        t.o_rdict = li.vf ? take(8 * t.ndict) : 0;
    }
    d.o_inv = take(8 * static_cast<int64_t>(rows_c) * nc);
    d.img_bytes = static_cast<int>(off);
    for (int q = 0; q + 1 < d.nlev; ++q) {  // vectors
        TailLevel &t = d.L[q];
        t.o_x = take(8 * (t.rows_per + t.gh_cap));
        t.o_t = take(8 * (t.rows_per + t.gh_cap));
        t.o_f = take(8 * t.rows_per);
        t.o_r = take(8 * t.rows_per);
    }
    {
        TailLevel &t = d.L[d.nlev - 1];
        t.n = nc;
        t.rows_per = rows_c;
        t.o_x = take(8 * rows_c);
        t.o_f = take(8 * rows_c);
    }
    d.o_fc = take(8 * nc);
    d.smem_bytes = static_cast<int>(off);
    if (off > budget) return;
    // per-CTA images
    std::vector<unsigned char> img(static_cast<size_t>(ctas) * d.img_bytes, 0);
    auto pack = [](int64_t j, int rp) { return static_cast<uint32_t>(((j / rp) << 16) | (j % rp)); };
    for (int r = 0; r < ctas; ++r) {
        unsigned char *b = img.data() + static_cast<size_t>(r) * d.img_bytes;
        auto *ngh = reinterpret_cast<int32_t *>(b);
        for (int q = 0; q + 1 < d.nlev; ++q) {
            const int k = k0 + q;
            const LevInfo &li = info[static_cast<size_t>(k)];
            const HostLevel &hl = H.levels[static_cast<size_t>(k)];
            const HostCsr &A = hl.A;
            const TailLevel &t = d.L[q];
            const int rpc = rows_per_of(k + 1);
            const int64_t r0 = std::min<int64_t>(A.n, static_cast<int64_t>(r) * t.rows_per);
            const int64_t r1 = std::min<int64_t>(A.n, static_cast<int64_t>(r + 1) * t.rows_per);
            const std::vector<int64_t> &g = li.ghosts[static_cast<size_t>(r)];
            ngh[q] = static_cast<int32_t>(g.size());
            auto *gh = reinterpret_cast<uint32_t *>(b + t.o_gh);
            for (size_t qg = 0; qg < g.size(); ++qg) gh[qg] = pack(g[qg], t.rows_per);
            auto *rp = reinterpret_cast<int32_t *>(b + t.o_rp);
            auto *col = reinterpret_cast<uint16_t *>(b + t.o_col);
            auto *agg = reinterpret_cast<uint32_t *>(b + t.o_agg);
            for (int64_t i = r0; i < r1; ++i) {
                const int64_t li_ = i - r0;
                rp[li_] = static_cast<int32_t>(A.rp[i] - A.rp[r0]);
                double dg = 0.0;
                for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
                    const int64_t le = e - A.rp[r0];
                    const int64_t j = A.ci[e];
                    col[le] = static_cast<uint16_t>(
                        (j >= r0 && j < r1) ? j - r0
                                            : t.rows_per + (std::lower_bound(g.begin(), g.end(), j) - g.begin()));
                    if (li.vf) {
                        uint64_t bits;
                        std::memcpy(&bits, &A.v[e], 8);
                        b[t.o_val + le] = static_cast<uint8_t>(li.ids.at(bits));
                        if (j == i) b[t.o_dix + li_] = static_cast<uint8_t>(li.ids.at(bits));
                    } else {
                        std::memcpy(b + t.o_val + 8 * le, &A.v[e], 8);
                    }
                    if (j == i) dg = A.v[e];
                }
                if (!li.vf) std::memcpy(b + t.o_dix + 8 * li_, &dg, 8);
                agg[li_] = pack(hl.agg[static_cast<size_t>(i)], rpc);
            }
            rp[r1 - r0] = static_cast<int32_t>(A.rp[r1] - A.rp[r0]);
            // members of the owned coarse rows (ascending fine rows)
            const int64_t ncl = (k + 1 == L - 1) ? nc : H.levels[static_cast<size_t>(k) + 1].A.n;
            const int64_t c0 = std::min<int64_t>(ncl, static_cast<int64_t>(r) * rpc);
            const int64_t c1 = std::min<int64_t>(ncl, static_cast<int64_t>(r + 1) * rpc);
            auto *mem = reinterpret_cast<uint32_t *>(b + t.o_mem);
            std::vector<int64_t> m0(static_cast<size_t>(c1 - c0), -1), m1(static_cast<size_t>(c1 - c0), -1);
            for (int64_t i = 0; i < A.n; ++i) {
                const int64_t p = hl.agg[static_cast<size_t>(i)];
                if (p < c0 || p >= c1) continue;
                auto &a = m0[static_cast<size_t>(p - c0)];
                if (a < 0) a = i;
                else m1[static_cast<size_t>(p - c0)] = i;
            }
            for (int64_t cc = c0; cc < c1; ++cc) {
                mem[2 * (cc - c0)] = pack(m0[static_cast<size_t>(cc - c0)], t.rows_per);
                const int64_t b1 = m1[static_cast<size_t>(cc - c0)];
                mem[2 * (cc - c0) + 1] = b1 < 0 ? 0xffffffffu : pack(b1, t.rows_per);
            }
            if (li.vf) {
                std::memcpy(b + t.o_dict, li.dict.data(), 8 * li.dict.size());
                for (size_t qd = 0; qd < li.dict.size(); ++qd) {
                    const double dv = std::fabs(li.dict[qd]);
                    const double y = (dv >= std::ldexp(1.0, -100) && dv <= std::ldexp(1.0, 100)) ? 1.0 / li.dict[qd] : 0.0;
                    std::memcpy(b + t.o_rdict + 8 * qd, &y, 8);
                }
            }
        }
        const int64_t c0 = std::min<int64_t>(nc, static_cast<int64_t>(r) * rows_c);
        const int64_t c1 = std::min<int64_t>(nc, static_cast<int64_t>(r + 1) * rows_c);
        std::memcpy(b + d.o_inv, H.inv.data() + c0 * nc, sizeof(double) * static_cast<size_t>((c1 - c0) * nc));
    }
    auto *dimg = dalloc<unsigned char>(c, static_cast<int64_t>(img.size()), true);
    CK(cudaMemcpy(dimg, img.data(), img.size(), cudaMemcpyHostToDevice));
    d.img = dimg;
    c->tail = dalloc<TailDesc>(c, 1, false);
    CK(cudaMemcpy(c->tail, &d, sizeof(d), cudaMemcpyHostToDevice));
    // the attribute is process-wide: leave it at the budget (never below what
    // another context's tail needs)
    CK(cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
    c->tail_ctas = ctas;
    c->tail_from = k0;
    c->tail_smem = d.smem_bytes;
    if (std::getenv("SB_TAIL_TRACE")) c->trace = dalloc<unsigned long long>(c, 256, false);
}

static std::string key_of(const char *kind, const Cyc *cp, const void *b, const void *x, const void *h) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s|%d|%d|%.17g|%p|%p|%p", kind, cp ? cp->pre : -1, cp ? cp->post : -1,
                  cp ? cp->omega : 0.0, b, x, h);
    return buf;
}

} // namespace sb

// ===========================================================================
// C ABI: context, solves, single kernels
// ===========================================================================
using namespace sb;

namespace sb {

static void destroy_graphs(sb_ctx c) {
    for (auto &kv : c->cache) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.g) cudaGraphDestroy(kv.second.g);
    }
    c->cache.clear();
}

static void ensure_hist(sb_ctx c, int need) {
    if (need <= c->hist_cap) return;
    destroy_graphs(c);  // graphs embed the history pointers
    const int cap = std::max(need, 1024);
    if (c->hist_r) cudaFree(c->hist_r);
    if (c->hist_t) cudaFree(c->hist_t);
    CK(cudaMalloc(&c->hist_r, sizeof(double) * cap));
    CK(cudaMalloc(&c->hist_t, sizeof(double) * cap));
    c->hist_cap = cap;
}

enum SolveKind { K_PCG = 0, K_BICG = 1, K_AMG = 2 };

// Runs the cached whole-solve graph (one launch, device-side loop control)
// and fills the report. host == true: b and x are host arrays and the H2D/D2H
// copies are part of the solve (the reference's wall_time covers its whole
// call, krylov.hpp:68,117).
static int run_solve(sb_ctx c, SolveKind kind, const sb_cycle *cpa, const double *b, double *x,
                     double tol, int max_iters, sb_report *rep, bool host, const char *who) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!(tol > 0.0)) throw invalid_argument(std::string(who) + ": tol must be > 0");
    Cyc cyc;
    const Cyc *cp = nullptr;
    if (cpa) {
        cyc = check_cycle(c, cpa, who);
        cp = &cyc;
    }
    if (kind == K_AMG && !cp) throw invalid_argument("amg_solve: cycle parameters required");
    CK(cudaSetDevice(c->device));
    const int64_t n = c->L[0].n;
    ensure_hist(c, std::max(max_iters, 0) + 2);
    const double *db = b;
    double *dx = x;
    if (host) {
        db = c->kv[KB];
        dx = c->kv[KX];
        CK(cudaMemcpyAsync(c->kv[KB], b, sizeof(double) * static_cast<size_t>(n), cudaMemcpyHostToDevice,
                           c->stream));
    }
    DevState hs;
    std::memset(&hs, 0, sizeof(hs));
    hs.tol = tol;
    hs.max_iters = max_iters;
    hs.hist_cap = c->hist_cap;
    hs.hist_r = c->hist_r;
    hs.hist_t = c->hist_t;
    CK(cudaMemcpyAsync(c->st, &hs, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
    const char *kname = kind == K_PCG ? "pcg" : kind == K_BICG ? "bicg" : "amg";
    auto build = [&]() {
        if (kind == K_PCG) return build_pcg(c, cp, db, dx);
        if (kind == K_BICG) return build_bicg(c, cp, db, dx);
        return build_amg(c, *cp, db, dx);
    };
    if (!c->graphs) {  // eager: the same kernels, host-side loop control
        CK(cudaEventRecord(c->ev0, c->stream));
        c->launch_count = 0;
        tl_eager = true;
        try {
            build();
        } catch (...) {
            tl_eager = false;
            throw;
        }
        tl_eager = false;
        c->last_launches = c->launch_count;
        CK(cudaEventRecord(c->ev1, c->stream));
    } else {
        const std::string key = key_of(kname, cp, db, dx, c->hist_r);
        auto it = c->cache.find(key);
        if (it == c->cache.end()) {
            GraphEntry e;
            c->plan = LaunchPlan{};
            e.g = build();
            e.plan = c->plan;
            CK(cudaGraphInstantiate(&e.exec, e.g, 0));
            it = c->cache.emplace(key, e).first;
        }
        CK(cudaEventRecord(c->ev0, c->stream));
        CK(cudaGraphLaunch(it->second.exec, c->stream));
        CK(cudaEventRecord(c->ev1, c->stream));
    }
    CK(cudaMemcpyAsync(&hs, c->st, sizeof(hs), cudaMemcpyDeviceToHost, c->stream));
    if (host)
        CK(cudaMemcpyAsync(x, dx, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->last_solve_ms = ms;
    if (c->graphs) {  // kernels the graph executed (LaunchPlan)
        const LaunchPlan &P = c->cache.find(key_of(kname, cp, db, dx, c->hist_r))->second.plan;
        const bool entered = hs.iter > 0 || kind == K_AMG;
        const int skipped = kind == K_BICG ? hs.half : (kind == K_PCG && hs.iter > 0 ? 1 : 0);
        c->last_launches = P.pre + P.post + (entered ? P.once : 0) + int64_t(hs.iter) * P.per_it +
                           std::max<int64_t>(0, int64_t(hs.iter) - skipped) * P.per_it_cond;
    }
    const int hist_len = hs.iter + 1;
    if (rep) {
        rep->iterations = hs.iter;
        rep->termination = hs.term;
        rep->true_residual = hs.true_res;
        rep->hist_len = hist_len;
        const int m = std::min(hist_len, std::max(rep->hist_cap, 0));
        if (m > 0 && rep->residual_history)
            CK(cudaMemcpy(rep->residual_history, c->hist_r, sizeof(double) * m, cudaMemcpyDeviceToHost));
        if (m > 0 && rep->time_history)
            CK(cudaMemcpy(rep->time_history, c->hist_t, sizeof(double) * m, cudaMemcpyDeviceToHost));
        rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (kind == K_AMG && hs.status == 2) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "amg_solve: diverged (residual %f exceeds 1e6 x initial %f)", hs.rn,
                      hs.r0);
        throw runtime_error(buf);
    }
    return SB_OK;
}

static const DevLevel &level_of(sb_ctx c, int k) {
    if (!c) throw invalid_argument("null context");
    if (k < 0 || k >= static_cast<int>(c->L.size())) throw invalid_argument("level out of range");
    return c->L[static_cast<size_t>(k)];
}

// Host-vector helper for the single-kernel entry points: copies in, runs fn
// on device buffers (scratch vectors of the context), copies out.
static void with_dev(sb_ctx c, const std::function<void(cudaStream_t)> &fn) {
    CK(cudaSetDevice(c->device));
    fn(c->stream);
    CK(cudaStreamSynchronize(c->stream));
}

static void h2d(sb_ctx c, double *d, const double *h, int64_t n) {
    CK(cudaMemcpyAsync(d, h, sizeof(double) * static_cast<size_t>(n), cudaMemcpyHostToDevice, c->stream));
}
static void d2h(sb_ctx c, double *h, const double *d, int64_t n) {
    CK(cudaMemcpyAsync(h, d, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, c->stream));
}

} // namespace sb

namespace sb {

// Context creation, split so the multi-rank path (sb_distrun.cuh) can upload
// partitioned levels in between.
static sb_ctx ctx_begin(const sb_device_opts &o) {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (o.device < 0 || o.device >= ndev) throw invalid_argument("sb_create: no such CUDA device");
    CK(cudaSetDevice(o.device));
    sb_ctx c = new sb_ctx_s;
    c->device = o.device;
    c->graphs = o.use_graphs != 0;
    if (const char *e = std::getenv("SB_PDL")) c->pdl = std::atoi(e) != 0;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    for (auto &s : c->cap) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return c;
}

// Launch configuration, coarse inverse, workspaces (n_vec = length of the
// Krylov / scratch vectors: n0, or own + ghost rows on a partitioned level 0),
// the cluster tail (only over levels >= tail_min).
static void ctx_finish(sb_ctx c, const Hier &h, const sb_device_opts &o, int64_t n_vec, int tail_min,
                       int64_t vec_headroom = 0) {
    size_t max_smem = 0;
    for (auto &l : c->L) max_smem = std::max({max_smem, l.smem, l.sell_smem, l.pat_tb,
                                               l.march_geo >= 0 ? march_smem_bytes(l.pat_tb, l.march_tb) : 0});
    if (max_smem > 200 * 1024) throw invalid_argument("sb_create: tile staging exceeds shared memory");
    {  // function attributes are process-wide: only ever raise them (a later
       // context with smaller tiles must not break an earlier one's launches)
        static std::mutex mu;
        static size_t raised = 0;
        std::lock_guard<std::mutex> lk(mu);
        max_smem = std::max(max_smem, raised);
        raised = max_smem;
    }
    set_smem_attr<M_SPMV, 0>(max_smem);
    set_smem_attr<M_SPMV, 1>(max_smem);
    set_smem_attr<M_SPMV, 2>(max_smem);
    set_smem_attr<M_RESID, 0>(max_smem);
    set_smem_attr<M_RESID, 1>(max_smem);
    set_smem_attr<M_JACOBI, 0>(max_smem);
    set_smem_attr<M_JACOBI, 1>(max_smem);
    set_smem_attr<M_JACOBI_PROLONG, 0>(max_smem);
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, o.device));
    for (auto &l : c->L) {
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_csr_tile<M_JACOBI, 0, 0, 0>, kTileRows, l.smem));
        l.grid = std::max(1, nsm * std::max(occ, 1));
        if (l.sell) {
            occ = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sellg<M_JACOBI, 0, 1, 1, 4, 0>, kTileRows,
                                                             l.sell_smem));
            l.sell_grid = std::max(1, nsm * std::max(occ, 1));
        }
        if (l.pat) {
            occ = 0;
            // resident CTAs of this level's kernel (wide rows: fewer, 1 row per thread)
            auto occ_of = [&](auto kern) {
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kPatThreads, l.pat_tb));
            };
            switch (l.pat_w) {
            case 16: occ_of(k_rowpat<M_JACOBI, 0, 16>); break;
            case 28: occ_of(k_rowpat<M_JACOBI, 0, 28>); break;
            case 32: occ_of(k_rowpat<M_JACOBI, 0, 32>); break;
            default: occ_of(k_rowpat<M_JACOBI, 0, 8>);
            }
            const int rows_it = kPatThreads * (l.pat_w <= 8 ? 2 : 1);
            const int64_t need = (l.n + rows_it - 1) / rows_it;
            l.pat_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, nsm * std::max(occ, 1))));
        }
        if (l.box_pair) {
            occ = 0;
            const int th = l.box_pair == 1 ? kBoxThreads : kCrossThreads;
            if (l.box_pair == 1)
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_boxpair<M_JACOBI, 0>, th, l.pat_tb));
            else if (l.pat_w == 7)
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_crosspair<M_JACOBI, 0, 7>, th, l.pat_tb));
            else
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_crosspair<M_JACOBI, 0, 5>, th, l.pat_tb));
            const int64_t need = (l.n / 2 + th - 1) / th;
            l.box_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, nsm * std::max(occ, 1))));
            l.box_grid_nv = l.box_grid;
            if (l.box_pair == 2) {
                occ = 0;
                if (l.pat_w == 7)
                    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_crosspair<M_SPMV, 1, 7>, th, l.pat_tb));
                else
                    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_crosspair<M_SPMV, 1, 5>, th, l.pat_tb));
                l.box_grid_nv =
                    static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, nsm * std::max(occ, 1))));
            }
        }
        if (l.march_geo >= 0) {
            occ = 0;
            const size_t sm = march_smem_bytes(l.pat_tb, l.march_tb);
            auto occ_m = [&](auto kern) {
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kMarchThreads, sm));
            };
#if SB_EXPERIMENTAL
            occ_m(k_march<M_JACOBI, 0, 0, 28, true>);
#else
            (void)occ_m;
#endif
            const int64_t need = std::max<int64_t>(l.march_ntiles, 1);
            l.march_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, nsm * std::max(occ, 1))));
        }
    }
    c->nc = h.nc;
    if (h.nc > 0) {
        c->alloc_host = c->host_from <= static_cast<int>(c->L.size()) - 1;  // the coarsest level's inverse
        c->inv = dalloc<double>(c, h.nc * h.nc);
        c->alloc_host = false;
        CK(cudaMemcpy(c->inv, h.inv.data(), sizeof(double) * h.inv.size(), cudaMemcpyHostToDevice));
        c->coarse_exact = o.coarse_exact != 0;
        if (c->coarse_exact) {
            c->lu = dalloc<double>(c, h.nc * h.nc);
            c->perm = dalloc<int32_t>(c, h.nc);
            CK(cudaMemcpy(c->lu, h.lu.data(), sizeof(double) * h.lu.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(c->perm, h.perm.data(), sizeof(int32_t) * h.perm.size(), cudaMemcpyHostToDevice));
        }
    }
    c->rs = dalloc<double>(c, n_vec);
    c->tail_min = tail_min;
    setup_tail(c, h);
    // Krylov vectors; on a partitioned level 0 in the window layout the halo
    // below own row 0 lives at negative indices (vec_headroom rows)
    for (auto &v : c->kv) v = dalloc<double>(c, vec_headroom + n_vec) + vec_headroom;
    int maxb = 148 * 8;  // reduction partials: one pair per CTA of any reducing kernel's grid
    for (auto &l : c->L)
        maxb = std::max({maxb, l.ntiles, l.grid, l.sell_grid, l.pat_grid, l.box_grid, l.march_grid});
    c->partials = dalloc<double>(c, 2 * static_cast<int64_t>(maxb) + 2, false);
    c->counter = dalloc<unsigned>(c, 4, false);
    c->st = dalloc<DevState>(c, 1, false);
    CK(cudaDeviceSynchronize());
}

} // namespace sb

extern "C" {

const char *sb_last_error(void) { return sb::g_err.c_str(); }
const char *sb_version(void) { return "sparsh_b200 0.1 (sm_100a)"; }

int sb_create(sb_hier hh, const sb_device_opts *opts, sb_ctx *out) {
    sb_ctx c = nullptr;
    int rc = guard([&] {
        Hier *h = hier_of(hh);
        if (!h || !out) throw invalid_argument("sb_create: null argument");
        sb_device_opts o{0, 1, -1, 0};
        if (opts) o = *opts;
        c = ctx_begin(o);
        const int64_t n0 = h->levels[0].A.n;
        const int L = static_cast<int>(h->levels.size());
        c->L.resize(h->levels.size());
        if (o.host_levels_from >= 0) c->host_from = static_cast<int>(std::min<int64_t>(o.host_levels_from, L));
        for (int k = 0; k < L; ++k)
            upload_level(c, h->levels[static_cast<size_t>(k)], c->L[static_cast<size_t>(k)], k + 1 == L, n0);
        // hybrid mode: no cluster tail (its shared-memory image would copy host levels to the device)
        ctx_finish(c, *h, o, n0, c->host_from < L ? L : 0);
        *out = c;
    });
    if (rc != SB_OK && c) sb_destroy(c);
    return rc;
}

void sb_destroy(sb_ctx c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    destroy_graphs(c);
    for (void *p : c->allocs) cudaFree(p);
    for (void *p : c->host_allocs) cudaFreeHost(p);
    if (c->hist_r) cudaFree(c->hist_r);
    if (c->hist_t) cudaFree(c->hist_t);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    for (auto &s : c->cap)
        if (s) cudaStreamDestroy(s);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int64_t sb_device_bytes(sb_ctx c) { return c ? c->bytes : 0; }
int64_t sb_host_bytes(sb_ctx c) { return c ? c->host_bytes : 0; }
void *sb_stream(sb_ctx c) { return c ? static_cast<void *>(c->stream) : nullptr; }

int sb_vcycle_dev(sb_ctx c, const sb_cycle *cp, int level, const double *d_f, double *d_x, int x_is_zero) {
    return guard([&] {
        level_of(c, level);
        const Cyc y = check_cycle(c, cp, "vcycle");
        CK(cudaSetDevice(c->device));
        emit_vcycle(c, c->stream, y, level, d_f, d_x, x_is_zero != 0);
    });
}

int sb_vcycle(sb_ctx c, const sb_cycle *cp, int level, const double *f, double *x) {
    return guard([&] {
        const DevLevel &l = level_of(c, level);
        const Cyc y = check_cycle(c, cp, "vcycle");
        double *df = c->kv[KB], *dx = c->kv[KX];
        bool zero = true;  // an all-zero initial guess takes the preconditioner path
        for (int64_t i = 0; i < l.n && zero; ++i) zero = (x[i] == 0.0 && !std::signbit(x[i]));
        with_dev(c, [&](cudaStream_t s) {
            h2d(c, df, f, l.n);
            h2d(c, dx, x, l.n);
            emit_vcycle(c, s, y, level, df, dx, zero);
            d2h(c, x, dx, l.n);
        });
    });
}

int sb_pcg(sb_ctx c, const sb_cycle *cp, const double *b, double *x, double tol, int max_iters,
           sb_report *rep) {
    return guard([&] { run_solve(c, K_PCG, cp, b, x, tol, max_iters, rep, true, "pcg"); });
}
int sb_pbicgstab(sb_ctx c, const sb_cycle *cp, const double *b, double *x, double tol, int max_iters,
                 sb_report *rep) {
    return guard([&] { run_solve(c, K_BICG, cp, b, x, tol, max_iters, rep, true, "pbicgstab"); });
}
int sb_amg_solve(sb_ctx c, const sb_cycle *cp, const double *b, double *x, double tol, int max_cycles,
                 sb_report *rep) {
    return guard([&] { run_solve(c, K_AMG, cp, b, x, tol, max_cycles, rep, true, "amg_solve"); });
}
int sb_pcg_dev(sb_ctx c, const sb_cycle *cp, const double *d_b, double *d_x, double tol, int max_iters,
               sb_report *rep) {
    return guard([&] { run_solve(c, K_PCG, cp, d_b, d_x, tol, max_iters, rep, false, "pcg"); });
}
int sb_pbicgstab_dev(sb_ctx c, const sb_cycle *cp, const double *d_b, double *d_x, double tol, int max_iters,
                     sb_report *rep) {
    return guard([&] { run_solve(c, K_BICG, cp, d_b, d_x, tol, max_iters, rep, false, "pbicgstab"); });
}

int64_t sb_last_solve_launches(sb_ctx c) { return c ? c->last_launches : 0; }
double sb_last_solve_ms(sb_ctx c) { return c ? c->last_solve_ms : 0.0; }

// Streamed storage of level k: fmt[0] = 2 row patterns / 1 sliced-ELL / 0 CSR, fmt[1] = value
// dictionary, fmt[2] = int16 column deltas, fmt[3] = slice width (max, padded
// to the group size);
// *matrix_bytes = bytes one pass over the matrix streams from HBM (entries
// incl. padding + per-row metadata), *nnz = stored nonzeros.
int sb_level_format(sb_ctx c, int k, int *fmt, int64_t *matrix_bytes, int64_t *nnz) {
    return guard([&] {
        const DevLevel &l = level_of(c, k);
        const int vb = l.vf ? 1 : 8, cb = l.cf ? 2 : 4;
        fmt[0] = l.pat ? 2 : l.sell;
        fmt[1] = l.vf;
        fmt[2] = l.cf;
        fmt[3] = l.pat ? l.pat_w : l.sell ? l.sell_ngmax * l.sell_gs : 0;
        if (l.pat) {
            *matrix_bytes = l.n + static_cast<int64_t>(l.pat_tb);  // 1 B/row + the table
        } else if (l.sell) {
            int64_t bytes = 0;  // every slice block is streamed once per pass
            CK(cudaMemcpy(&bytes, l.soff + l.sell_tiles, sizeof(int64_t), cudaMemcpyDeviceToHost));
            *matrix_bytes = bytes;
        } else {
            *matrix_bytes = l.nnz * (vb + cb) + 4 * (l.n + 1);
        }
        *nnz = l.nnz;
    });
}

int sb_build_flags(void) { return kExperimental ? 1 : 0; }

int sb_level_residency(sb_ctx c, int k, int *on_host, int64_t *matrix_bytes) {
    return guard([&] {
        const DevLevel &l = level_of(c, k);
        if (on_host) *on_host = k >= c->host_from ? 1 : 0;
        if (matrix_bytes) {
            int fmt[4];
            int64_t nnz = 0;
            const int rc = sb_level_format(c, k, fmt, matrix_bytes, &nnz);
            if (rc != SB_OK) throw runtime_error(sb_last_error());
        }
        (void)l;
    });
}

int sb_level_fused_sweeps(sb_ctx c, int k, int *geo) {
    try {
        const DevLevel &l = level_of(c, k);
        if (geo && l.tb == 1) {
            const TbGeo &g = l.tb_geo;
            const int v[8] = {g.nx, g.ny, g.nz, g.TX, g.TY, g.ZL, l.tb_grid, static_cast<int>(l.tb_smem)};
            std::memcpy(geo, v, sizeof v);
        } else if (geo && l.tb == 2) {
            const BoxGeo &g = l.box_geo;
            const int v[8] = {g.nx, g.ny, g.nz, l.box_tx, l.box_tx >= 16 ? 8 : 16, 8, l.tb_grid,
                              static_cast<int>(box2_smem(l.box_tx))};
            std::memcpy(geo, v, sizeof v);
        }
        return l.tb ? 2 : 1;
    } catch (const std::exception &e) {
        set_error(e.what());
        return -1;
    }
}

int sb_level_sweep_kernel(sb_ctx c, int k, char *buf, int cap) {
    return guard([&] {
        const DevLevel &l = level_of(c, k);
        if (!buf || cap < 1) throw invalid_argument("sb_level_sweep_kernel: no buffer");
        const char *name = l.pat ? (l.box_pair == 1 ? "k_boxpair" : l.box_pair == 2 ? "k_crosspair"
                                    : l.march_geo >= 0 ? "k_march" : "k_rowpat")
                                 : l.sell ? "k_sellg" : "k_csr_tile";
        std::snprintf(buf, static_cast<size_t>(cap), "%s", name);
    });
}

int sb_level_march(sb_ctx c, int k, int *geo, int *stride) {
    return guard([&] {
        const DevLevel &l = level_of(c, k);
        *geo = l.march_geo;
        *stride = l.march_S;
    });
}

// Diagnostics: copies the tail kernel's phase timestamps (SB_TAIL_TRACE=1) into
// out (count first); returns the number of entries, or -1 if tracing is off.
int sb_tail_trace(sb_ctx c, unsigned long long *out, int cap) {
    if (!c || !c->trace) return -1;
    unsigned long long buf[256];
    if (cudaMemcpy(buf, c->trace, sizeof(buf), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    const int n = static_cast<int>(std::min<unsigned long long>(buf[0], 255));
    for (int i = 0; i < n && i < cap; ++i) out[i] = buf[1 + i];
    return n;
}
int sb_tail_info(sb_ctx c, int *tail_from, int *ctas, int *smem) {
    if (!c) return SB_EINVAL;
    *tail_from = c->tail_from;
    *ctas = c->tail_ctas;
    *smem = c->tail_smem;
    return SB_OK;
}

int sb_vcycle_launches(sb_ctx c, const sb_cycle *cp) {
    int out = 0;
    const int rc = guard([&] {
        const Cyc y = check_cycle(c, cp, "vcycle");
        // count by a dry emission into a throw-away capture
        cudaGraph_t g = begin_capture(c);
        c->launch_count = 0;
        emit_vcycle(c, c->stream, y, 0, c->kv[KB], c->kv[KX], true);
        out = c->launch_count;
        end_capture(c, g);
        cudaGraphDestroy(g);
    });
    return rc == SB_OK ? out : -1;
}

static int time_kernel(sb_ctx c, int kind, int level, const sb_cycle *cp, int reps, int64_t flush_bytes,
                       double *avg_ms, int *launches) {
    return guard([&] {
        const DevLevel &l = level_of(c, level);
        if (reps < 1) throw invalid_argument("sb_time_kernel: reps must be >= 1");
        Cyc y;
        if (kind == 0 || kind == 3 || kind == 4 || kind == 5) y = check_cycle(c, cp, "sb_time_kernel");
        CK(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        double *x = c->kv[KX], *t = c->kv[KZ], *f = c->kv[KB];
        k_fill<<<vec_grid(l.n), kVecThreads, 0, s>>>(l.n, f, 1.0);
        k_fill<<<vec_grid(l.n), kVecThreads, 0, s>>>(l.n, x, 0.5);
        k_fill<<<vec_grid(l.n), kVecThreads, 0, s>>>(l.n, t, 0.5);
        CK(cudaGetLastError());
        cudaGraphExec_t vgraph = nullptr;
        int vlaunch = 0;
        auto once = [&]() {
            c->launch_count = 0;
            if (kind == 0) {
                launch_jacobi(c, l, s, x, f, t, y.omega);
                std::swap(x, t);
            } else if (kind == 1) {
                launch_csr<M_SPMV, 0>(c, l, s, x, nullptr, t, 0.0, nullptr, Red{});
            } else if (kind == 2) {
                launch_csr<M_RESID, 0>(c, l, s, x, f, t, 0.0, nullptr, Red{});
            } else if (kind == 3) {
                emit_vcycle(c, s, y, level, f, t, true);
            } else if (kind == 4) {
                if (!vgraph) {
                    cudaGraph_t g = begin_capture(c);
                    c->launch_count = 0;
                    emit_vcycle(c, s, y, level, f, t, true);
                    vlaunch = c->launch_count;
                    end_capture(c, g);
                    CK(cudaGraphInstantiate(&vgraph, g, 0));
                    cudaGraphDestroy(g);
                }
                CK(cudaGraphLaunch(vgraph, s));
                c->launch_count = vlaunch;
            } else if (kind == 5) {  // 32 chained Jacobi sweeps captured as one graph
                if (!vgraph) {
                    cudaGraph_t g = begin_capture(c);
                    c->launch_count = 0;
                    for (int r = 0; r < 32; ++r) {
                        launch_jacobi(c, l, s, x, f, t, y.omega);
                        std::swap(x, t);
                    }
                    vlaunch = c->launch_count;
                    end_capture(c, g);
                    CK(cudaGraphInstantiate(&vgraph, g, 0));
                    cudaGraphDestroy(g);
                }
                CK(cudaGraphLaunch(vgraph, s));
                c->launch_count = vlaunch;
            } else {
                throw invalid_argument("sb_time_kernel: unknown kind");
            }
        };
        once();  // warm-up
        float ms = 0.f;
        if (flush_bytes <= 0) {
            CK(cudaEventRecord(c->ev0, s));
            for (int i = 0; i < reps; ++i) once();
            CK(cudaEventRecord(c->ev1, s));
            CK(cudaEventSynchronize(c->ev1));
            CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        } else {
            // cold L2: a write of flush_bytes (> L2) before every launch, each
            // launch bracketed by its own event pair on the launching stream
            double *fb = nullptr;
            CK(cudaMalloc(&fb, static_cast<size_t>(flush_bytes)));
            struct Free {
                double *p;
                ~Free() { cudaFree(p); }
            } free_fb{fb};
            const int64_t nf = flush_bytes / 8;
            for (int i = 0; i < reps; ++i) {
                k_fill<<<vec_grid(nf), kVecThreads, 0, s>>>(nf, fb, static_cast<double>(i));
                CK(cudaEventRecord(c->ev0, s));
                once();
                CK(cudaEventRecord(c->ev1, s));
                CK(cudaEventSynchronize(c->ev1));
                float one = 0.f;
                CK(cudaEventElapsedTime(&one, c->ev0, c->ev1));
                ms += one;
            }
        }
        if (avg_ms) *avg_ms = ms / reps;
        if (launches) *launches = c->launch_count;
        if (vgraph) cudaGraphExecDestroy(vgraph);
    });
}

#ifdef SB_XP_TRACE
extern "C" int sb_debug_xp_trace(unsigned long long *out, int cap, int reset) {
    unsigned n = 0;
    cudaMemcpyFromSymbol(&n, g_xp_n, sizeof(n));
    n = std::min<unsigned>(n, 65536u);
    const int m = std::min<int>(static_cast<int>(n), cap);
    if (m > 0) cudaMemcpyFromSymbol(out, g_xp_trace, sizeof(unsigned long long) * 6 * m);
    if (reset) {
        unsigned z = 0;
        cudaMemcpyToSymbol(g_xp_n, &z, sizeof(z));
    }
    return m;
}
#endif
int sb_time_kernel(sb_ctx c, int kind, int level, const sb_cycle *cp, int reps, double *avg_ms, int *launches) {
    return time_kernel(c, kind, level, cp, reps, 0, avg_ms, launches);
}

int sb_time_kernel_cold(sb_ctx c, int kind, int level, const sb_cycle *cp, int reps, int64_t flush_bytes,
                        double *avg_ms, int *launches) {
    if (flush_bytes <= 0)
        return guard([] { throw invalid_argument("sb_time_kernel_cold: flush_bytes must be > 0"); });
    return time_kernel(c, kind, level, cp, reps, flush_bytes, avg_ms, launches);
}

int sb_spmv(sb_ctx c, int level, const double *x, double *y) {
    return guard([&] {
        const DevLevel &l = level_of(c, level);
        with_dev(c, [&](cudaStream_t s) {
            h2d(c, c->kv[KP], x, l.n);
            launch_csr<M_SPMV, 0>(c, l, s, c->kv[KP], nullptr, c->kv[KAP], 0.0, nullptr, Red{});
            d2h(c, y, c->kv[KAP], l.n);
        });
    });
}

int sb_smooth(sb_ctx c, int level, const sb_cycle *cp, double *x, const double *f, int sweeps) {
    return guard([&] {
        const DevLevel &l = level_of(c, level);
        if (sweeps < 0) throw invalid_argument("smooth: negative sweep count");
        if (!cp || cp->smoother != SB_SMOOTHER_JACOBI)
            throw invalid_argument("smooth: only the weighted Jacobi smoother runs on the device");
        if (!(cp->omega > 0.0) || cp->omega > 1.0)
            throw invalid_argument("SmootherKind: Jacobi weight " + std::to_string(cp->omega) +
                                   " outside (0, 1]");
        if (sweeps == 0) return;
        if (l.bad_diag >= 0)
            throw invalid_argument("smooth: zero diagonal entry in row " + std::to_string(l.bad_diag));
        with_dev(c, [&](cudaStream_t s) {
            double *a = c->kv[KX], *b = c->kv[KZ], *df = c->kv[KB];
            h2d(c, a, x, l.n);
            h2d(c, df, f, l.n);
            emit_sweeps(c, l, s, sweep_groups(l, sweeps, false), a, b, df, cp->omega);
            d2h(c, x, a, l.n);
        });
    });
}

int sb_residual(sb_ctx c, int level, const double *x, const double *f, double *r) {
    return guard([&] {
        const DevLevel &l = level_of(c, level);
        with_dev(c, [&](cudaStream_t s) {
            h2d(c, c->kv[KX], x, l.n);
            h2d(c, c->kv[KB], f, l.n);
            launch_csr<M_RESID, 0>(c, l, s, c->kv[KX], c->kv[KB], c->kv[KR], 0.0, nullptr, Red{});
            d2h(c, r, c->kv[KR], l.n);
        });
    });
}

int sb_restrict(sb_ctx c, int level, const double *r, double *fc) {
    return guard([&] {
        const DevLevel &l = level_of(c, level);
        if (l.nc < 0) throw invalid_argument("restrict: coarsest level has no aggregation");
        with_dev(c, [&](cudaStream_t s) {
            h2d(c, c->kv[KR], r, l.n);
            k_restrict<<<vec_grid(l.nc), kVecThreads, 0, s>>>(l.nc, l.mem, c->kv[KR], c->kv[KZ], nullptr, nullptr, 0.0);
            CK(cudaGetLastError());
            d2h(c, fc, c->kv[KZ], l.nc);
        });
    });
}

int sb_prolong(sb_ctx c, int level, const double *xc, double *x) {
    return guard([&] {
        const DevLevel &l = level_of(c, level);
        if (l.nc < 0) throw invalid_argument("prolong: coarsest level has no aggregation");
        with_dev(c, [&](cudaStream_t s) {
            h2d(c, c->kv[KZ], xc, l.nc);
            h2d(c, c->kv[KX], x, l.n);
            k_prolong<<<vec_grid(l.n), kVecThreads, 0, s>>>(l.n, l.agg, c->kv[KX], c->kv[KZ], c->kv[KX]);
            CK(cudaGetLastError());
            d2h(c, x, c->kv[KX], l.n);
        });
    });
}

int sb_coarse_solve(sb_ctx c, const double *f, double *x) {
    return guard([&] {
        if (!c || c->nc <= 0) throw invalid_argument("coarse_solve: no coarse factorization");
        with_dev(c, [&](cudaStream_t s) {
            h2d(c, c->kv[KB], f, c->nc);
            emit_coarse(c, s, c->kv[KB], c->kv[KX]);
            d2h(c, x, c->kv[KX], c->nc);
        });
    });
}

} // extern "C"

#include "sb_distrun.cuh"
