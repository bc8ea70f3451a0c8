/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the solve phase.
 *
 * A plain-C restatement of the reference (sparsh, /root/reference/proj) for
 * the hot path named by BASELINE.json: CSR SpMV, weighted-Jacobi smoothing,
 * residual, unit-P restriction/prolongation, dense-LU coarse solve, the
 * V-cycle, PCG, flexible PBiCGStab and the stationary AMG solve, plus the
 * host setup that feeds it (node-HEM aggregation, Galerkin product). Each
 * function cites the reference file:line it restates; evaluation order and
 * rounding follow the reference exactly (build with -O3 -ffp-contract=off),
 * so results are bit-identical to the reference compiled the same way —
 * tests/test_oracle.py pins that against oracle/_ref and tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. The product (paper_2007_00056_b200) never does.
 *
 * Paths: inc/ = /root/reference/proj/include/sparsh/.
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define OC_MAX_LEVELS 64

typedef struct {
    int32_t n, ncols;
    int64_t nnz;
    int32_t *rp; /* n+1 */
    int32_t *ci; /* nnz */
    double *v;   /* nnz */
} oc_csr;

typedef struct {
    int iterations;
    int termination; /* inc/convergence.hpp:15 order: converged, max_iters, breakdown, diverged */
    double wall_time;
    double true_residual;
    int hist_len;
    int hist_cap;
    double *residual_history;
    double *time_history;
} oc_report;

enum { OC_CONVERGED = 0, OC_MAX_ITERS = 1, OC_BREAKDOWN = 2, OC_DIVERGED = 3 };

typedef struct {
    int nlevels;
    int stalled;
    oc_csr A[OC_MAX_LEVELS];
    int32_t *agg[OC_MAX_LEVELS]; /* fine_to_coarse of level k (k < nlevels-1) */
    int32_t nc[OC_MAX_LEVELS];
    double *lu;    /* dense row-major LU of the coarsest level */
    int32_t *perm; /* row permutation */
    int pre, post;
    double omega;
} oc_hier;

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ---- L1: inc/csr.hpp ---------------------------------------------------- */

/* inc/csr.hpp:174-194 — y_i = sum_k val_k * x[col_k], sequential from 0.0. */
void oc_spmv(const oc_csr *A, const double *x, double *y) {
    for (int32_t i = 0; i < A->n; ++i) {
        double sum = 0.0;
        for (int32_t k = A->rp[i]; k < A->rp[i + 1]; ++k) sum += A->v[k] * x[A->ci[k]];
        y[i] = sum;
    }
}

/* Dot-product summation order. 0 (default): the reference's sequential sum
 * (inc/csr.hpp:245-251). 1: a reordered sum -- sequential within blocks of 256
 * products, then a pairwise tree over the block sums -- used only to measure
 * how far a legal reordering of the reference's own dots moves a solve (the
 * rounding-noise floor of the parity contract; tools/noise_floor.py). */
static int g_dot_mode = 0;
void oc_set_dot_mode(int mode) { g_dot_mode = mode; }

static double dot_tree(int64_t n, const double *a, const double *b) {
    if (n <= 256) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    }
    int64_t h = ((n + 511) / 512) * 256; /* split at a block boundary */
    return dot_tree(h, a, b) + dot_tree(n - h, a + h, b + h);
}

/* inc/csr.hpp:245-251 */
double oc_dot(int64_t n, const double *a, const double *b) {
    if (g_dot_mode == 1) return dot_tree(n, a, b);
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
/* inc/csr.hpp:253 */
double oc_norm2(int64_t n, const double *a) { return sqrt(oc_dot(n, a, a)); }
/* inc/csr.hpp:256-260 — y += alpha x */
static void oc_axpy(int64_t n, double alpha, const double *x, double *y) {
    for (int64_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}

/* inc/csr.hpp:267-274 — r = f - A x (spmv first, then subtract). */
void oc_residual(const oc_csr *A, const double *x, const double *f, double *r) {
    oc_spmv(A, x, r);
    for (int32_t i = 0; i < A->n; ++i) r[i] = f[i] - r[i];
}

/* inc/csr.hpp:226-241 with P = prolongation_from_aggregation (inc/aggregation.hpp:68-82):
 * one unit entry per row, so y[agg[i]] += 1.0 * r[i] in ascending i. */
void oc_restrict(int32_t n, const int32_t *agg, int32_t nc, const double *r, double *fc) {
    for (int32_t c = 0; c < nc; ++c) fc[c] = 0.0;
    for (int32_t i = 0; i < n; ++i) fc[agg[i]] += 1.0 * r[i];
}

/* inc/cycle.hpp:72-73: correction = spmv(P, x_c) (0.0 + 1.0*x_c), then axpy(1.0, correction, x). */
void oc_prolong_add(int32_t n, const int32_t *agg, const double *xc, double *x) {
    for (int32_t i = 0; i < n; ++i) {
        double corr = 0.0;
        corr += 1.0 * xc[agg[i]];
        x[i] += 1.0 * corr;
    }
}

/* ---- smoother: inc/smoother.hpp ----------------------------------------- */

/* inc/smoother.hpp:55-70 — diagonal position per row; returns the first bad
 * row (missing or zero diagonal) or -1. */
static int32_t oc_diag_positions(const oc_csr *A, int32_t *pos) {
    for (int32_t i = 0; i < A->n; ++i) {
        int32_t lo = A->rp[i], hi = A->rp[i + 1];
        while (lo < hi) { /* lower_bound */
            int32_t mid = lo + (hi - lo) / 2;
            if (A->ci[mid] < i) lo = mid + 1; else hi = mid;
        }
        if (lo == A->rp[i + 1] || A->ci[lo] != i || A->v[lo] == 0.0) return i;
        pos[i] = lo;
    }
    return -1;
}

/* inc/smoother.hpp:95-123 (Jacobi branch :109-121): per sweep Ax = spmv(A, x),
 * then x_i += omega * (f_i - Ax_i) / a_ii. Returns -1, or the bad-diagonal row. */
int32_t oc_jacobi(const oc_csr *A, double omega, double *x, const double *f, int sweeps) {
    if (sweeps == 0) return -1;
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(A->n > 0 ? A->n : 1));
    const int32_t bad = oc_diag_positions(A, pos);
    if (bad >= 0) { free(pos); return bad; }
    double *Ax = (double *)malloc(sizeof(double) * (size_t)(A->n > 0 ? A->n : 1));
    for (int s = 0; s < sweeps; ++s) {
        oc_spmv(A, x, Ax);
        for (int32_t i = 0; i < A->n; ++i) {
            const double aii = A->v[pos[i]];
            x[i] += omega * (f[i] - Ax[i]) / aii;
        }
    }
    free(Ax);
    free(pos);
    return -1;
}

/* ---- setup: inc/coarsen.hpp, inc/aggregation.hpp ------------------------ */

/* inc/coarsen.hpp:31-73 (ascending visit, alternate_ends = false): pair with the
 * unassigned neighbour of largest |a_ij| (strict >, stored zeros skipped),
 * coarse ids in discovery order. Returns n_coarse. */
int32_t oc_node_hem(const oc_csr *A, int32_t *f2c) {
    int32_t next = 0;
    for (int32_t i = 0; i < A->n; ++i) f2c[i] = -1;
    for (int32_t i = 0; i < A->n; ++i) {
        if (f2c[i] >= 0) continue;
        int32_t best = -1;
        double bw = 0.0;
        for (int32_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            const int32_t j = A->ci[k];
            if (j == i || f2c[j] >= 0) continue;
            const double w = fabs(A->v[k]);
            if (w != 0.0 && (best < 0 || w > bw)) { best = j; bw = w; }
        }
        f2c[i] = next;
        if (best >= 0) f2c[best] = next;
        ++next;
    }
    return next;
}

static int cmp_i32(const void *a, const void *b) {
    const int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* inc/aggregation.hpp:92-152 — per coarse row k: members ascending, entries in
 * CSR order, accumulate into a dense SPA; touched columns sorted; every touched
 * entry stored (even an exact 0.0 sum). Allocates out's arrays. */
void oc_galerkin(const oc_csr *A, const int32_t *f2c, int32_t nc, oc_csr *out) {
    const int32_t n = A->n;
    int32_t *mptr = (int32_t *)calloc((size_t)nc + 1, sizeof(int32_t));
    int32_t *mem = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t *next = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nc > 0 ? nc : 1));
    for (int32_t i = 0; i < n; ++i) ++mptr[f2c[i] + 1];
    for (int32_t c = 0; c < nc; ++c) mptr[c + 1] += mptr[c];
    for (int32_t c = 0; c < nc; ++c) next[c] = mptr[c];
    for (int32_t i = 0; i < n; ++i) mem[next[f2c[i]]++] = i;

    double *acc = (double *)calloc((size_t)(nc > 0 ? nc : 1), sizeof(double));
    char *touched = (char *)calloc((size_t)(nc > 0 ? nc : 1), 1);
    int32_t *here = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nc > 0 ? nc : 1));
    int64_t cap = A->nnz > 0 ? A->nnz : 1, cnt = 0;
    out->rp = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nc + 1));
    out->ci = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    out->v = (double *)malloc(sizeof(double) * (size_t)cap);
    out->rp[0] = 0;
    for (int32_t k = 0; k < nc; ++k) {
        int32_t nh = 0;
        for (int32_t m = mptr[k]; m < mptr[k + 1]; ++m) {
            const int32_t i = mem[m];
            for (int32_t e = A->rp[i]; e < A->rp[i + 1]; ++e) {
                const int32_t l = f2c[A->ci[e]];
                if (!touched[l]) { touched[l] = 1; here[nh++] = l; }
                acc[l] += A->v[e];
            }
        }
        qsort(here, (size_t)nh, sizeof(int32_t), cmp_i32);
        for (int32_t t = 0; t < nh; ++t) {
            const int32_t l = here[t];
            out->ci[cnt] = l;
            out->v[cnt] = acc[l];
            ++cnt;
            acc[l] = 0.0;
            touched[l] = 0;
        }
        out->rp[k + 1] = (int32_t)cnt;
    }
    out->n = out->ncols = nc;
    out->nnz = cnt;
    free(mptr); free(mem); free(next); free(acc); free(touched); free(here);
}

/* ---- coarse solve: inc/coarse_solver.hpp ------------------------------- */

/* inc/coarse_solver.hpp:129-166 — dense LU with partial pivoting (first max
 * |a_ik| wins, strict >), singular when pivot == 0 or |pivot| < 1e-14 max|a|.
 * Returns -1 or the singular row. */
int32_t oc_dense_lu(const oc_csr *A, double *lu, int32_t *perm) {
    const size_t n = (size_t)A->n;
    double max_abs = 0.0;
    memset(lu, 0, sizeof(double) * n * n);
    for (int32_t i = 0; i < A->n; ++i)
        for (int32_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            lu[(size_t)i * n + (size_t)A->ci[k]] = A->v[k];
            if (fabs(A->v[k]) > max_abs) max_abs = fabs(A->v[k]);
        }
    for (size_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
    const double tol = 1e-14 * max_abs;
    for (size_t k = 0; k < n; ++k) {
        size_t p = k;
        for (size_t i = k + 1; i < n; ++i)
            if (fabs(lu[i * n + k]) > fabs(lu[p * n + k])) p = i;
        const double pivot = lu[p * n + k];
        if (pivot == 0.0 || fabs(pivot) < tol) return (int32_t)k;
        if (p != k) {
            for (size_t j = 0; j < n; ++j) {
                const double t = lu[p * n + j];
                lu[p * n + j] = lu[k * n + j];
                lu[k * n + j] = t;
            }
            const int32_t t = perm[p]; perm[p] = perm[k]; perm[k] = t;
        }
        for (size_t i = k + 1; i < n; ++i) {
            const double m = lu[i * n + k] / pivot;
            lu[i * n + k] = m;
            for (size_t j = k + 1; j < n; ++j) lu[i * n + j] -= m * lu[k * n + j];
        }
    }
    return -1;
}

/* inc/coarse_solver.hpp:168-182 — permuted forward then backward substitution. */
void oc_dense_solve(int32_t n_, const double *lu, const int32_t *perm, const double *b, double *y) {
    const size_t n = (size_t)n_;
    for (size_t i = 0; i < n; ++i) {
        double s = b[perm[i]];
        for (size_t j = 0; j < i; ++j) s -= lu[i * n + j] * y[j];
        y[i] = s;
    }
    for (size_t i = n; i-- > 0;) {
        double s = y[i];
        for (size_t j = i + 1; j < n; ++j) s -= lu[i * n + j] * y[j];
        y[i] = s / lu[i * n + i];
    }
}

/* ---- hierarchy: inc/hierarchy.hpp:51-76 --------------------------------- */

static void csr_copy(const oc_csr *src, oc_csr *dst) {
    dst->n = src->n;
    dst->ncols = src->ncols;
    dst->nnz = src->nnz;
    dst->rp = (int32_t *)malloc(sizeof(int32_t) * ((size_t)src->n + 1));
    dst->ci = (int32_t *)malloc(sizeof(int32_t) * (size_t)(src->nnz > 0 ? src->nnz : 1));
    dst->v = (double *)malloc(sizeof(double) * (size_t)(src->nnz > 0 ? src->nnz : 1));
    memcpy(dst->rp, src->rp, sizeof(int32_t) * ((size_t)src->n + 1));
    memcpy(dst->ci, src->ci, sizeof(int32_t) * (size_t)src->nnz);
    memcpy(dst->v, src->v, sizeof(double) * (size_t)src->nnz);
}

void oc_hier_free(oc_hier *h) {
    if (!h) return;
    for (int k = 0; k < h->nlevels; ++k) {
        free(h->A[k].rp); free(h->A[k].ci); free(h->A[k].v);
        free(h->agg[k]);
    }
    free(h->lu);
    free(h->perm);
    free(h);
}

/* Builds the node-HEM hierarchy (coarsening = node_hem, coarse_solver = direct).
 * Returns NULL with *err = 1 (coarse dim > 2000: the reference's sparse-LU path,
 * not restated) or 2 (singular coarse pivot). */
oc_hier *oc_hier_build(const oc_csr *A0, int32_t coarse_target, int max_levels, int *err) {
    oc_hier *h = (oc_hier *)calloc(1, sizeof(oc_hier));
    *err = 0;
    h->pre = h->post = 6;
    h->omega = 2.0 / 3.0;
    csr_copy(A0, &h->A[0]);
    h->nlevels = 1;
    while (h->A[h->nlevels - 1].n > coarse_target && h->nlevels < max_levels &&
           h->nlevels < OC_MAX_LEVELS) {
        oc_csr *Af = &h->A[h->nlevels - 1];
        int32_t *f2c = (int32_t *)malloc(sizeof(int32_t) * (size_t)(Af->n > 0 ? Af->n : 1));
        const int32_t nc = oc_node_hem(Af, f2c);
        if (nc == Af->n) { free(f2c); h->stalled = 1; break; }
        oc_galerkin(Af, f2c, nc, &h->A[h->nlevels]);
        h->agg[h->nlevels - 1] = f2c;
        h->nc[h->nlevels - 1] = nc;
        h->nlevels++;
    }
    const oc_csr *Ac = &h->A[h->nlevels - 1];
    if (Ac->n > 2000) { *err = 1; oc_hier_free(h); return NULL; }
    h->lu = (double *)malloc(sizeof(double) * (size_t)Ac->n * (size_t)Ac->n + 8);
    h->perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)Ac->n + 4);
    if (oc_dense_lu(Ac, h->lu, h->perm) >= 0) { *err = 2; oc_hier_free(h); return NULL; }
    return h;
}

int oc_hier_nlevels(const oc_hier *h) { return h->nlevels; }
const oc_csr *oc_hier_level(const oc_hier *h, int k) { return &h->A[k]; }
const int32_t *oc_hier_agg(const oc_hier *h, int k) { return h->agg[k]; }
void oc_hier_set_cycle(oc_hier *h, int pre, int post, double omega) {
    h->pre = pre; h->post = post; h->omega = omega;
}
void oc_coarse_solve(const oc_hier *h, const double *f, double *x) {
    oc_dense_solve(h->A[h->nlevels - 1].n, h->lu, h->perm, f, x);
}

/* ---- V-cycle: inc/cycle.hpp:53-75 --------------------------------------- */

/* Returns -1 or a bad-diagonal row. */
int32_t oc_vcycle(const oc_hier *h, int k, const double *f, double *x) {
    const oc_csr *A = &h->A[k];
    if (k + 1 == h->nlevels) { oc_coarse_solve(h, f, x); return -1; }
    int32_t bad = oc_jacobi(A, h->omega, x, f, h->pre);
    if (bad >= 0) return bad;
    const int32_t n = A->n, nc = h->nc[k];
    double *r = (double *)malloc(sizeof(double) * (size_t)n);
    double *fc = (double *)malloc(sizeof(double) * (size_t)nc);
    double *xc = (double *)calloc((size_t)nc, sizeof(double));
    oc_residual(A, x, f, r);
    oc_restrict(n, h->agg[k], nc, r, fc);
    bad = oc_vcycle(h, k + 1, fc, xc);
    if (bad < 0) {
        oc_prolong_add(n, h->agg[k], xc, x);
        bad = oc_jacobi(A, h->omega, x, f, h->post);
    }
    free(r); free(fc); free(xc);
    return bad;
}

static void oc_precond(const oc_hier *h, int32_t n, const double *r, double *z) {
    if (!h) { memcpy(z, r, sizeof(double) * (size_t)n); return; }
    memset(z, 0, sizeof(double) * (size_t)n); /* inc/cycle.hpp:140-144: z = zeros; one cycle */
    oc_vcycle(h, 0, r, z);
}

static void rec(oc_report *rep, double value, double t0) {
    if (rep->hist_len < rep->hist_cap) {
        if (rep->residual_history) rep->residual_history[rep->hist_len] = value;
        if (rep->time_history) rep->time_history[rep->hist_len] = now_s() - t0;
    }
    rep->hist_len++;
}

/* ---- Krylov: inc/krylov.hpp --------------------------------------------- */

/* inc/krylov.hpp:65-119 */
void oc_pcg(const oc_csr *A, const oc_hier *h, const double *b, double *x, double tol,
            int max_iters, oc_report *rep) {
    const double t0 = now_s();
    const int32_t n = A->n;
    const size_t sz = sizeof(double) * (size_t)(n > 0 ? n : 1);
    double *r = (double *)malloc(sz), *z = (double *)malloc(sz), *p = (double *)malloc(sz),
           *Ap = (double *)malloc(sz);
    rep->hist_len = 0;
    rep->iterations = 0;
    rep->termination = OC_MAX_ITERS;
    memset(x, 0, sz);
    memcpy(r, b, sizeof(double) * (size_t)n);
    double rn = oc_norm2(n, r);
    const double r0 = rn;
    rec(rep, rn, t0);
    if (rn < tol) {
        rep->termination = OC_CONVERGED;
    } else {
        oc_precond(h, n, r, z);
        memcpy(p, z, sizeof(double) * (size_t)n);
        double rz = oc_dot(n, r, z);
        for (int j = 0; j < max_iters; ++j) {
            oc_spmv(A, p, Ap);
            const double pAp = oc_dot(n, Ap, p);
            if (pAp <= 0.0) { rep->termination = OC_BREAKDOWN; break; }
            const double alpha = rz / pAp;
            oc_axpy(n, alpha, p, x);
            oc_axpy(n, -alpha, Ap, r);
            rn = oc_norm2(n, r);
            rec(rep, rn, t0);
            rep->iterations = j + 1;
            if (rn < tol) { rep->termination = OC_CONVERGED; break; }
            if (rn > 1e6 * r0) { rep->termination = OC_DIVERGED; break; }
            oc_precond(h, n, r, z);
            const double rz_next = oc_dot(n, r, z);
            const double beta = rz_next / rz;
            rz = rz_next;
            for (int32_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        }
    }
    oc_residual(A, x, b, r);
    rep->true_residual = oc_norm2(n, r);
    rep->wall_time = now_s() - t0;
    free(r); free(z); free(p); free(Ap);
}

/* inc/krylov.hpp:126-211 — flexible PBiCGStab, rbar0 = r0, p = r + beta(p - omega Ap~). */
void oc_pbicgstab(const oc_csr *A, const oc_hier *h, const double *b, double *x, double tol,
                  int max_iters, oc_report *rep) {
    const double eps = 1e-300;
    const double t0 = now_s();
    const int32_t n = A->n;
    const size_t sz = sizeof(double) * (size_t)(n > 0 ? n : 1);
    double *r = (double *)malloc(sz), *rbar = (double *)malloc(sz), *p = (double *)malloc(sz),
           *pt = (double *)malloc(sz), *Apt = (double *)malloc(sz), *s = (double *)malloc(sz),
           *st = (double *)malloc(sz), *Ast = (double *)malloc(sz);
    rep->hist_len = 0;
    rep->iterations = 0;
    rep->termination = OC_MAX_ITERS;
    memset(x, 0, sz);
    memcpy(r, b, sizeof(double) * (size_t)n);
    double rn = oc_norm2(n, r);
    const double r0 = rn;
    rec(rep, rn, t0);
    if (rn < tol) {
        rep->termination = OC_CONVERGED;
    } else {
        memcpy(rbar, r, sizeof(double) * (size_t)n);
        memcpy(p, r, sizeof(double) * (size_t)n);
        double rho = oc_dot(n, r, rbar);
        for (int j = 0; j < max_iters; ++j) {
            if (fabs(rho) < eps) { rep->termination = OC_BREAKDOWN; break; }
            oc_precond(h, n, p, pt);
            oc_spmv(A, pt, Apt);
            const double denom = oc_dot(n, Apt, rbar);
            if (fabs(denom) < eps) { rep->termination = OC_BREAKDOWN; break; }
            const double alpha = rho / denom;
            memcpy(s, r, sizeof(double) * (size_t)n);
            oc_axpy(n, -alpha, Apt, s);
            const double sn = oc_norm2(n, s);
            if (sn < tol) {
                oc_axpy(n, alpha, pt, x);
                rec(rep, sn, t0);
                rep->iterations = j + 1;
                rep->termination = OC_CONVERGED;
                break;
            }
            oc_precond(h, n, s, st);
            oc_spmv(A, st, Ast);
            const double AsAs = oc_dot(n, Ast, Ast);
            if (AsAs < eps) { rep->termination = OC_BREAKDOWN; break; }
            const double omega = oc_dot(n, Ast, s) / AsAs;
            oc_axpy(n, alpha, pt, x);
            oc_axpy(n, omega, st, x);
            memcpy(r, s, sizeof(double) * (size_t)n);
            oc_axpy(n, -omega, Ast, r);
            rn = oc_norm2(n, r);
            rec(rep, rn, t0);
            rep->iterations = j + 1;
            if (rn < tol) { rep->termination = OC_CONVERGED; break; }
            if (rn > 1e6 * r0) { rep->termination = OC_DIVERGED; break; }
            if (fabs(omega) < eps) { rep->termination = OC_BREAKDOWN; break; }
            const double rho_next = oc_dot(n, r, rbar);
            const double beta = (rho_next / rho) * (alpha / omega);
            rho = rho_next;
            for (int32_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * Apt[i]);
        }
    }
    oc_residual(A, x, b, r);
    rep->true_residual = oc_norm2(n, r);
    rep->wall_time = now_s() - t0;
    free(r); free(rbar); free(p); free(pt); free(Apt); free(s); free(st); free(Ast);
}

/* inc/cycle.hpp:91-130 — returns 0, or 2 on divergence (the reference throws
 * runtime_error "amg_solve: diverged ..."). */
int oc_amg_solve(const oc_hier *h, const double *b, double *x, double tol, int max_cycles,
                 oc_report *rep) {
    const double t0 = now_s();
    const oc_csr *A = &h->A[0];
    const int32_t n = A->n;
    double *r = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    rep->hist_len = 0;
    rep->iterations = 0;
    rep->termination = OC_MAX_ITERS;
    memset(x, 0, sizeof(double) * (size_t)n);
    double rn = oc_norm2(n, b);
    const double r0 = rn;
    int status = 0;
    rec(rep, rn, t0);
    if (rn < tol) rep->termination = OC_CONVERGED;
    for (int c = 1; rep->termination != OC_CONVERGED && c <= max_cycles; ++c) {
        oc_vcycle(h, 0, b, x);
        oc_residual(A, x, b, r);
        rn = oc_norm2(n, r);
        rec(rep, rn, t0);
        rep->iterations = c;
        if (rn > 1e6 * r0) { status = 2; break; }
        if (rn < tol) rep->termination = OC_CONVERGED;
    }
    rep->true_residual = rn;
    rep->wall_time = now_s() - t0;
    free(r);
    return status;
}
