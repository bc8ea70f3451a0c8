/*
 * sparsh_b200.h — C ABI of the B200-native solve phase (libsparsh_b200.so).
 *
 * Drop-in boundary for the reference's solve-phase API (sparsh, C++20,
 * /root/reference/proj/include/sparsh). Each entry point cites the reference
 * interface it replaces; INTEGRATION.md shows the binding a maintainer adds.
 * Plain pointers and sizes only: no C++ or torch types cross this boundary.
 *
 * Status codes (every int-returning call):
 *   SB_OK       0  success
 *   SB_EINVAL   1  the reference would throw std::invalid_argument
 *   SB_ERUNTIME 2  the reference would throw std::runtime_error
 *                  (amg_solve divergence, singular coarse pivot)
 *   SB_ECUDA    3  CUDA / NCCL failure (no CPU fallback exists)
 * sb_last_error() returns the thread-local message of the last failure,
 * phrased like the reference's exception text ("diverged", "zero diagonal
 * entry in row i", ...).
 *
 * Threading: a built hierarchy (sb_hier) is immutable and shareable. A device
 * context (sb_ctx) owns mutable device workspaces and CUDA graphs, so one
 * context serves one solve at a time (the one deviation from the reference's
 * "concurrent V-cycles are safe"). Termination codes equal the
 * reference enum order (inc/convergence.hpp:15).
 */
#ifndef SPARSH_B200_H
#define SPARSH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB_OK 0
#define SB_EINVAL 1
#define SB_ERUNTIME 2
#define SB_ECUDA 3

/* inc/convergence.hpp:15 */
#define SB_CONVERGED 0
#define SB_MAX_ITERS 1
#define SB_BREAKDOWN 2
#define SB_DIVERGED 3

/* inc/smoother.hpp:23-28 — only weighted Jacobi runs on the device; the
 * Gauss-Seidel families are rejected with SB_EINVAL (no CPU emulation). */
#define SB_SMOOTHER_JACOBI 0
#define SB_SMOOTHER_GS_FORWARD 1
#define SB_SMOOTHER_GS_BACKWARD 2
#define SB_SMOOTHER_GS_SYMMETRIC 3

/* Host CSR matrix, borrowed. Mirrors sparsh::CsrMatrix (inc/csr.hpp:44-169):
 * int32 column indices strictly increasing per row, f64 values. Row offsets
 * are int32 (the reference's index_t, inc/csr.hpp:22; zero-copy from a
 * CsrMatrix) or int64 (for nnz > INT32_MAX): set exactly one of the two. */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    const int32_t *row_ptr32;
    const int64_t *row_ptr64;
    const int32_t *col_idx;
    const double *values;
} sb_csr;

/* inc/config.hpp:81-105 (setup subset). coarsening: 0 node_hem (1 edge_hem is
 * rejected); coarse_solver: 0 direct (1 cg is rejected on the device path;
 * -1 = no coarse factorization, for identity-preconditioned cg/bicgstab only). */
typedef struct {
    int coarsening;
    int64_t coarse_target;
    int max_levels;
    int coarse_solver;
    int threads; /* host threads for the Galerkin product (0 = all) */
    int galerkin_gpu; /* 1: Galerkin products A_c = P^T A P on the GPU (bit-identical; north star (c)) */
    int gpu_device;   /* CUDA ordinal used when galerkin_gpu = 1 */
} sb_setup_opts;

/* inc/cycle.hpp:24-32 (CycleParams) */
typedef struct {
    int pre_sweeps;
    int post_sweeps;
    int smoother; /* SB_SMOOTHER_* */
    double omega; /* Jacobi weight, (0, 1] (inc/smoother.hpp:33-38) */
} sb_cycle;

/* inc/convergence.hpp:33-42 (ConvergenceReport). The caller owns the history
 * buffers (hist_cap entries each, may be NULL); hist_len is the reference's
 * residual_history.size() (= iterations + 1), even when > hist_cap. */
typedef struct {
    int iterations;
    int termination;
    double wall_time;
    double true_residual;
    int hist_len;
    int hist_cap;
    double *residual_history;
    double *time_history;
} sb_report;

/* Device-context options. */
typedef struct {
    int device;          /* CUDA ordinal */
    int use_graphs;      /* 1: whole-solve CUDA graph with device-side loop control (default);
                            0: eager launches on sb_stream, host-side loop control (same kernels,
                            same bits; one host sync per conditional decision) */
    int64_t host_levels_from; /* hybrid mode (paper's MI scheme): the matrix storage of levels
                                 >= this index stays in pinned host memory and the device
                                 kernels read it over the host link (zero-copy; no CPU
                                 compute); -1 = all levels device-resident */
    int coarse_exact;    /* 0: coarsest solve = GEMV with the precomputed inverse (fast);
                            1: the reference's permuted forward/backward substitution in
                               its exact operation order (bit-identical, slow; parity mode) */
} sb_device_opts;

typedef struct sb_hier_s *sb_hier;
typedef struct sb_ctx_s *sb_ctx;

const char *sb_last_error(void);
const char *sb_version(void);

/* ---- host setup: bit-exact with the reference ---------------------------- */

/* sparsh::Hierarchy(CsrMatrix, SolverConfig) — inc/hierarchy.hpp:51-76:
 * node-HEM (inc/coarsen.hpp:31-73) + Galerkin (inc/aggregation.hpp:92-152)
 * until n <= coarse_target or max_levels, then the dense LU of the coarsest
 * level (inc/coarse_solver.hpp:129-166; > 2000 rows -> SB_EINVAL, the sparse
 * LU path is not provided). Deep-copies A. */
int sb_setup(const sb_csr *A, const sb_setup_opts *opts, sb_hier *out);
/* galerkin_product(A, agg) — inc/aggregation.hpp:92-152 — computed on CUDA
 * device `device`: bit-identical to the reference (one thread per coarse row
 * replays the reference's accumulation order). Aggregates must have 1 or 2
 * fine nodes (node-HEM). *out is malloc'ed: free with sb_free_csr. */
int sb_galerkin_gpu(const sb_csr *A, const int32_t *fine_to_coarse, int64_t n_coarse, int device, sb_csr *out);
/* Adopt a hierarchy built elsewhere (e.g. by the reference itself): levels[k]
 * and fine_to_coarse[k] (k < nlevels-1) exactly as sparsh::Level holds them
 * (inc/hierarchy.hpp:24-28). The coarse LU is factorized here. */
int sb_hier_from_levels(int nlevels, const sb_csr *levels, const int32_t *const *fine_to_coarse,
                        sb_hier *out);
void sb_hier_free(sb_hier h);
int sb_hier_nlevels(sb_hier h);                        /* Hierarchy::nlevels, :78 */
int sb_hier_stalled(sb_hier h);                        /* Hierarchy::coarsening_stalled, :82 */
/* Borrowed views of level k (valid while h lives): A (row_ptr32 set when it fits),
 * the aggregation (NULL on the coarsest level), n_coarse (-1 on the coarsest). */
int sb_hier_level(sb_hier h, int k, sb_csr *A, const int32_t **fine_to_coarse, int64_t *n_coarse);
/* Coarse factorization counters (inc/coarse_solver.hpp:75-77). */
int sb_hier_coarse_counts(sb_hier h, long *symbolic, long *numeric, long *solves);

/* ---- device context --------------------------------------------------------- */

/* Upload every level (CSR, diagonal, aggregate maps) plus the coarse inverse
 * to the device; allocate workspaces; record graphs lazily per sb_cycle. */
int sb_create(sb_hier h, const sb_device_opts *opts, sb_ctx *out);
void sb_destroy(sb_ctx ctx);
/* Device bytes resident for the hierarchy (paper's memory metric). */
int64_t sb_device_bytes(sb_ctx ctx);
/* Hybrid mode: bytes of level storage kept in pinned host memory (levels >=
 * host_levels_from and, when the coarsest level is among them, its inverse). */
int64_t sb_host_bytes(sb_ctx ctx);
/* The CUDA stream the context launches on (cudaStream_t as void*). */
void *sb_stream(sb_ctx ctx);

/* ---- solve phase (the hot path) ------------------------------------------- */

/* vcycle_in_place(h, k, f, x, p) — inc/cycle.hpp:53-75. Host vectors of level
 * k's size; x_is_zero promises x == 0 on entry (the preconditioner case,
 * inc/cycle.hpp:140-144). */
int sb_vcycle(sb_ctx ctx, const sb_cycle *cp, int level, const double *f, double *x);
/* Same on device pointers (stream-ordered on sb_stream). */
int sb_vcycle_dev(sb_ctx ctx, const sb_cycle *cp, int level, const double *d_f, double *d_x,
                  int x_is_zero);

/* pcg(A, b, make_amg_preconditioner(h, cp), tol, max_iters) — inc/krylov.hpp:65-119
 * with inc/cycle.hpp:137-145. A is level 0 of the context. cp == NULL selects
 * Preconditioner::identity() (inc/krylov.hpp:33-35), i.e. cg(). tol is the
 * reference's ABSOLUTE tolerance. x receives the solution. */
int sb_pcg(sb_ctx ctx, const sb_cycle *cp, const double *b, double *x, double tol,
           int max_iters, sb_report *rep);
/* pbicgstab(...) — inc/krylov.hpp:126-211 (flexible; cp == NULL -> bicgstab()). */
int sb_pbicgstab(sb_ctx ctx, const sb_cycle *cp, const double *b, double *x, double tol,
                 int max_iters, sb_report *rep);
/* amg_solve(h, b, tol, max_cycles, p) — inc/cycle.hpp:91-130. Divergence ->
 * SB_ERUNTIME ("amg_solve: diverged ..."), report still filled. */
int sb_amg_solve(sb_ctx ctx, const sb_cycle *cp, const double *b, double *x, double tol,
                 int max_cycles, sb_report *rep);
/* Device-pointer variants (inputs already resident; the bench's kernel-only number). */
int sb_pcg_dev(sb_ctx ctx, const sb_cycle *cp, const double *d_b, double *d_x, double tol,
               int max_iters, sb_report *rep);
int sb_pbicgstab_dev(sb_ctx ctx, const sb_cycle *cp, const double *d_b, double *d_x,
                     double tol, int max_iters, sb_report *rep);

/* ---- measurement --------------------------------------------------------- */

/* CUDA-event time (ms) of the last whole-solve graph launch on sb_stream. */
double sb_last_solve_ms(sb_ctx ctx);
/* Kernels the last solve executed on the device (graph mode: counted from the
 * captured graph's structure and the iteration count; eager mode: launched). */
int64_t sb_last_solve_launches(sb_ctx ctx);
/* Times `reps` back-to-back launches of one kernel on level `level` with CUDA
 * events on sb_stream; *avg_ms = mean per launch. kind: 0 Jacobi sweep,
 * 1 SpMV, 2 residual, 3 one V-cycle from x = 0 launched eagerly, 4 the same
 * V-cycle captured once as a CUDA graph and replayed, 5 a graph of 32 chained
 * Jacobi sweeps (the in-graph cost of one sweep = *avg_ms / *launches; cp
 * required for 0, 3, 4, 5). *launches = kernels launched per repetition. */
int sb_time_kernel(sb_ctx ctx, int kind, int level, const sb_cycle *cp, int reps, double *avg_ms,
                   int *launches);
/* Same, with a cold L2: before every launch a write of flush_bytes (> the
 * 126 MB L2) on sb_stream, and one event pair around each launch. */
int sb_time_kernel_cold(sb_ctx ctx, int kind, int level, const sb_cycle *cp, int reps, int64_t flush_bytes,
                        double *avg_ms, int *launches);
/* Diagnostics: tail-kernel phase timestamps (needs SB_TAIL_TRACE=1 at
 * sb_create) and the tail placement (first tail level, cluster CTAs, smem). */
int sb_tail_trace(sb_ctx ctx, unsigned long long *out, int cap);
int sb_tail_info(sb_ctx ctx, int *tail_from, int *ctas, int *smem_bytes);
/* Streamed storage of level k (lossless): fmt = {sliced-ELL?, value dictionary?,
 * int16 column deltas?, slice width}; *matrix_bytes = HBM bytes one matrix pass
 * streams (entries incl. padding + per-row metadata); *nnz = stored nonzeros. */
int sb_level_format(sb_ctx ctx, int level, int *fmt, int64_t *matrix_bytes, int64_t *nnz);
/* Plane-marching sweep of a row-pattern level (sb_march.cuh, opt-in with
 * SB_MARCH=1): *geo = -1 (none) or 0 (27-point box); *stride = plane stride. */
int sb_level_march(sb_ctx ctx, int level, int *geo, int *stride);
/* Name of the kernel a Jacobi sweep of `level` launches (k_boxpair, k_march,
 * k_rowpat, k_sellg or k_csr_tile), NUL-terminated into buf[cap]. */
int sb_level_sweep_kernel(sb_ctx ctx, int level, char *buf, int cap);
/* Jacobi sweeps one HBM pass performs on level k: 2 when consecutive sweeps
 * run fused in k_cross_tb2 (temporal blocking on structured 7-point levels),
 * else 1; -1 on error. geo (8 ints, optional) receives {nx, ny, nz, TX, TY,
 * ZL, grid, smem bytes} of the fused kernel. */
int sb_level_fused_sweeps(sb_ctx ctx, int level, int *geo);
/* Build flags of the library: bit 0 = built with SB_EXPERIMENTAL=1 (the
 * kernels kept for A/B work: k_march, k_cross_rr, k_cross_tb2). */
int sb_build_flags(void);
/* Placement of level k's matrix storage (hybrid mode, sb_device_opts.host_levels_from):
 * *on_host = 1 when it lives in pinned host memory, *matrix_bytes = its streamed
 * bytes (as sb_level_format). Compare with the reference's analytical model
 * (inc/memory_model.hpp: csr_bytes, plan_mi / plan_ci). */
int sb_level_residency(sb_ctx ctx, int level, int *on_host, int64_t *matrix_bytes);
/* Kernels launched by one V-cycle from level 0 (graph node count). */
int sb_vcycle_launches(sb_ctx ctx, const sb_cycle *cp);

/* ---- single kernels on a level (unit parity; host vectors) --------------- */

/* spmv(A_k, x, y) — inc/csr.hpp:174-194 */
int sb_spmv(sb_ctx ctx, int level, const double *x, double *y);
/* smooth_in_place(jacobi, A_k, x, f, sweeps) — inc/smoother.hpp:95-123 */
int sb_smooth(sb_ctx ctx, int level, const sb_cycle *cp, double *x, const double *f, int sweeps);
/* residual(A_k, x, f) — inc/csr.hpp:267-274 */
int sb_residual(sb_ctx ctx, int level, const double *x, const double *f, double *r);
/* spmv_transpose(P_k, r) — inc/csr.hpp:226-241, inc/cycle.hpp:69 */
int sb_restrict(sb_ctx ctx, int level, const double *r, double *f_coarse);
/* x += spmv(P_k, x_c) — inc/cycle.hpp:72-73 */
int sb_prolong(sb_ctx ctx, int level, const double *x_coarse, double *x);
/* CoarseFactorization::solve — inc/coarse_solver.hpp:63-71 */
int sb_coarse_solve(sb_ctx ctx, const double *f, double *x);

/* ---- multi-GPU row partition --------------------------------- */

/* Rank `rank` of `nranks`: contiguous owned rows per distributed level (level 0
 * split evenly, coarse levels induced by the aggregates), columns renumbered
 * [own | ghost] or kept as global offsets in the window layout (info11[9..10] = rows
 * below / above own in the x vectors), exchange plans (recv_dst: where each peer's
 * chunk lands relative to own row 0) for the x halo, straddling-aggregate residuals
 * and coarse parents; levels with < gather_rows rows (and below) replicated.
 * Host-only; every rank computes identical plans from the same hierarchy. */
typedef struct sb_part_s *sb_part;
int sb_partition(sb_hier h, int rank, int nranks, int64_t gather_rows, sb_part *out);
void sb_partition_free(sb_part p);
int sb_partition_info(sb_part p, int *nlevels, int *first_replicated);
int sb_partition_level(sb_part p, int level, int64_t *info11, sb_csr *A_local, const int64_t **ghost,
                       const int64_t **rghost, const int64_t **xcghost, const int32_t **mem0,
                       const int32_t **mem1, const int32_t **parent);
int sb_partition_exchange(sb_part p, int level, int which, int64_t *counts4, const int **send_peers,
                          const int64_t **send_off, const int32_t **send_idx, const int **recv_peers,
                          const int64_t **recv_off, const int64_t **recv_dst);

/* Partitioned solve. NCCL mode: one rank per process/GPU; rank 0 calls
 * sb_nccl_unique_id and broadcasts the 128 bytes (e.g. torch.distributed);
 * b / x are the rank's own rows [lo, hi) (sb_dist_rows). In-process mode
 * (sb_dist_create_local): nranks virtual ranks on one device sharing this
 * process (exchanges are peer-buffer gathers) — b / x are global vectors.
 * Same termination semantics and report as sb_pcg / sb_pbicgstab; the
 * V-cycle is bitwise identical to the single-GPU one. */
typedef struct sb_dist_s *sb_dist;
int sb_nccl_unique_id(unsigned char *out128);
int sb_dist_create(sb_hier h, int rank, int nranks, const unsigned char *nccl_id128, int64_t gather_rows,
                   const sb_device_opts *opts, sb_dist *out);
int sb_dist_create_local(sb_hier h, int nranks, int64_t gather_rows, const sb_device_opts *opts,
                         sb_dist *out);
/* Peer-memory (P2P) transport instead of NCCL: halo / straddle / gather
 * exchanges are gathers straight out of the peers' own rows, dot products sum
 * every rank's partials in rank order; ordering through per-rank epoch
 * counters in peer-visible memory (publish after the producing kernels, one
 * spinning thread waits for the peers). One rank per process:
 * sb_dist_create_p2p, then sb_dist_p2p_export (CUDA IPC handles of the
 * buffers peers read; call with buf = NULL for the length), exchange the blobs
 * out of band, sb_dist_p2p_connect with every rank's blob in rank order
 * (len_each bytes apart). sb_dist_create_local_p2p: nranks in-process ranks on
 * one device over the same protocol (tests). */
int sb_dist_create_p2p(sb_hier h, int rank, int nranks, int64_t gather_rows, const sb_device_opts *opts,
                       sb_dist *out);
int sb_dist_p2p_export(sb_dist d, unsigned char *buf, int64_t cap, int64_t *len);
int sb_dist_p2p_connect(sb_dist d, const unsigned char *blobs, int64_t len_each);
int sb_dist_create_local_p2p(sb_hier h, int nranks, int64_t gather_rows, const sb_device_opts *opts,
                             sb_dist *out);
void sb_dist_destroy(sb_dist d);
int sb_dist_rows(sb_dist d, int local_rank, int64_t *lo, int64_t *hi, int *first_replicated);
int sb_dist_pcg(sb_dist d, const sb_cycle *cp, const double *b, double *x, double tol, int max_iters,
                sb_report *rep, int device_ptrs);
int sb_dist_pbicgstab(sb_dist d, const sb_cycle *cp, const double *b, double *x, double tol,
                      int max_iters, sb_report *rep, int device_ptrs);
int sb_dist_vcycle(sb_dist d, const sb_cycle *cp, const double *f, double *x);
double sb_dist_last_solve_ms(sb_dist d);   /* CUDA-event time of the last solve, max over hosted ranks */
int sb_dist_last_launches(sb_dist d);      /* kernels rank 0 of this process launched in it */

/* ---- problem generators (harness inputs) ------------------- */

/* convdiff2d(nx, ny, bx, by, c) — inc/problems.hpp:28-57, bit-identical.
 * Arrays allocated with malloc; free with sb_free_csr. */
int sb_gen_convdiff2d(int64_t nx, int64_t ny, double bx, double by, double c, sb_csr *out);
/* 3D 7-point: diag, and off-diagonals (x-, x+, y-, y+, z-, z+). */
int sb_gen_stencil7(int64_t nx, int64_t ny, int64_t nz, double diag, const double off[6],
                    sb_csr *out);
/* 3D 7-point upwind convection-diffusion, cell-volume scaled like convdiff2d. */
int sb_gen_convdiff3d(int64_t nx, int64_t ny, int64_t nz, double bx, double by, double bz,
                      double c, sb_csr *out);
/* 3D 27-point: diag, -1 to every neighbour (times off). */
int sb_gen_stencil27(int64_t nx, int64_t ny, int64_t nz, double diag, double off, sb_csr *out);
/* sb_setup of the 27-point operator generated straight into the hierarchy's
 * host storage (no intermediate copies: config 5, 512^3 with nnz 3.6e9 > int32,
 * is set up in ~50 GB of host memory). Identical to sb_gen_stencil27 + sb_setup. */
int sb_setup_stencil27(int64_t nx, int64_t ny, int64_t nz, double diag, double off, const sb_setup_opts *opts,
                       sb_hier *out);
void sb_free_csr(sb_csr *m);
/* read_matrix_market(path) — inc/mm_io.hpp:35-111 (coordinate real general |
 * symmetric; duplicates summed as the reference's from_triplets, csr.hpp:57-95).
 * I/O and format errors -> SB_ERUNTIME with the reference's messages. Free with
 * sb_free_csr. */
int sb_read_matrix_market(const char *path, sb_csr *out);
/* write_matrix_market(A, path) — inc/mm_io.hpp:114-135 (general, 1-based, %.17g). */
int sb_write_matrix_market(const char *path, const sb_csr *A);
/* rhs_random(n, seed) — inc/problems.hpp:69-75 (std::mt19937, U[0,1)), bit-identical. */
int sb_gen_rhs_random(int64_t n, unsigned seed, double *out);

#ifdef __cplusplus
}
#endif
#endif
