// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// C-ABI driver over the UNMODIFIED reference headers (sparsh, header-only
// C++20) compiled where they lie under /root/reference/proj/include. It
// exists so tests/ and bench.py's CPU-baseline leg can run the reference's
// own code through ctypes. Built by oracle/Makefile into
// oracle/_ref/libsparsh_ref.so with the reference's canonical flags
// (-O3 -ffp-contract=off: the reference's CMake sets no -march, so no FMA;
// see SURVEY.md §8c). No reference source is copied into this repository.
//
// Every entry point returns 0 on success, 1 for std::invalid_argument, 2 for
// std::runtime_error (message via ref_last_error()).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparsh/sparsh.hpp"

using namespace sparsh;

namespace {
thread_local std::string g_err;

template <typename Fn> int guard(Fn &&fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error &e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 2;
    }
}

struct RefHier {
    std::unique_ptr<Hierarchy> h;
    CycleParams cp;
};

CycleParams make_cp(int family, double omega, int pre, int post) {
    CycleParams cp;
    cp.pre_sweeps = pre;
    cp.post_sweeps = post;
    switch (family) {
    case 0: cp.smoother = SmootherKind::weighted_jacobi(omega); break;
    case 1: cp.smoother = SmootherKind::gauss_seidel_forward(); break;
    case 2: cp.smoother = SmootherKind::gauss_seidel_backward(); break;
    default: cp.smoother = SmootherKind::gauss_seidel_symmetric(); break;
    }
    return cp;
}

DenseVector vec(const double *p, std::int64_t n) { return DenseVector(p, p + n); }
} // namespace

extern "C" {

typedef struct {
    int iterations;
    int termination;
    double wall_time;
    double true_residual;
    int hist_len;
    int hist_cap;
    double *residual_history;
    double *time_history;
} ref_report;

const char *ref_last_error(void) { return g_err.c_str(); }
void ref_set_threads(unsigned n) { set_thread_count(n); }
unsigned ref_get_threads(void) { return thread_count(); }

// ---- matrices -------------------------------------------------------------
int ref_csr_new(int32_t nrows, int32_t ncols, const int32_t *rp, const int32_t *ci,
                const double *v, void **out) {
    return guard([&] {
        const std::int64_t nnz = rp[nrows];
        *out = new CsrMatrix(nrows, ncols, std::vector<index_t>(rp, rp + nrows + 1),
                             std::vector<index_t>(ci, ci + nnz),
                             std::vector<double>(v, v + nnz));
    });
}
int ref_csr_from_triplets(int32_t nrows, int32_t ncols, int64_t ntrip, const int32_t *r,
                          const int32_t *c, const double *v, void **out) {
    return guard([&] {
        std::vector<Triplet> t(static_cast<std::size_t>(ntrip));
        for (int64_t k = 0; k < ntrip; ++k) t[k] = {r[k], c[k], v[k]};
        *out = new CsrMatrix(CsrMatrix::from_triplets(nrows, ncols, std::move(t)));
    });
}
int ref_convdiff2d(int32_t nx, int32_t ny, double bx, double by, double c, void **out) {
    return guard([&] { *out = new CsrMatrix(convdiff2d(nx, ny, bx, by, c)); });
}
// 3D generators for the BASELINE configs, built the way the
// reference's own 2D generators are (inc/problems.hpp:28-57): triplets of
// (row, col, value) into CsrMatrix::from_triplets (inc/csr.hpp:57-95), which
// sorts the columns and stores 0.0 + value. Node m = (iz*ny + iy)*nx + ix,
// Dirichlet boundaries (out-of-grid neighbours dropped). These are test
// infrastructure: bench.py's reference arm and tests/golden/make_config_fixtures.py
// build their matrices here, so no product library is loaded on that path.
// off = {x-, x+, y-, y+, z-, z+}.
int ref_stencil7(int32_t nx, int32_t ny, int32_t nz, double diag, const double *off, void **out) {
    return guard([&] {
        if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("stencil7: grid dims must be >= 1");
        const index_t n = nx * ny * nz;
        std::vector<Triplet> e;
        e.reserve(7 * static_cast<std::size_t>(n));
        for (index_t iz = 0; iz < nz; ++iz)
            for (index_t iy = 0; iy < ny; ++iy)
                for (index_t ix = 0; ix < nx; ++ix) {
                    const index_t m = (iz * ny + iy) * nx + ix;
                    e.push_back({m, m, diag});
                    if (ix > 0) e.push_back({m, m - 1, off[0]});
                    if (ix < nx - 1) e.push_back({m, m + 1, off[1]});
                    if (iy > 0) e.push_back({m, m - nx, off[2]});
                    if (iy < ny - 1) e.push_back({m, m + nx, off[3]});
                    if (iz > 0) e.push_back({m, m - nx * ny, off[4]});
                    if (iz < nz - 1) e.push_back({m, m + nx * ny, off[5]});
                }
        *out = new CsrMatrix(CsrMatrix::from_triplets(n, n, std::move(e)));
    });
}
// -lap(u) + b.grad(u) + c u on (0,1)^3, first-order upwinding scaled by the
// cell volume: convdiff2d's expressions (inc/problems.hpp:34-41) extended to z.
int ref_convdiff3d(int32_t nx, int32_t ny, int32_t nz, double bx, double by, double bz, double c,
                   void **out) {
    const double hx = 1.0 / (static_cast<double>(nx) + 1.0);
    const double hy = 1.0 / (static_cast<double>(ny) + 1.0);
    const double hz = 1.0 / (static_cast<double>(nz) + 1.0);
    const double ax = hy * hz / hx, ay = hx * hz / hy, az = hx * hy / hz;
    const double diag = 2.0 * (ax + ay + az) + std::abs(bx) * hy * hz + std::abs(by) * hx * hz +
                        std::abs(bz) * hx * hy + c * hx * hy * hz;
    const double off[6] = {-ax - std::max(bx, 0.0) * hy * hz, -ax + std::min(bx, 0.0) * hy * hz,
                           -ay - std::max(by, 0.0) * hx * hz, -ay + std::min(by, 0.0) * hx * hz,
                           -az - std::max(bz, 0.0) * hx * hy, -az + std::min(bz, 0.0) * hx * hy};
    return ref_stencil7(nx, ny, nz, diag, off, out);
}
// 27-point box stencil (diag, `off` to all 26 neighbours).
int ref_stencil27(int32_t nx, int32_t ny, int32_t nz, double diag, double off, void **out) {
    return guard([&] {
        if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("stencil27: grid dims must be >= 1");
        const index_t n = nx * ny * nz;
        std::vector<Triplet> e;
        e.reserve(27 * static_cast<std::size_t>(n));
        for (index_t iz = 0; iz < nz; ++iz)
            for (index_t iy = 0; iy < ny; ++iy)
                for (index_t ix = 0; ix < nx; ++ix) {
                    const index_t m = (iz * ny + iy) * nx + ix;
                    for (int dz = -1; dz <= 1; ++dz)
                        for (int dy = -1; dy <= 1; ++dy)
                            for (int dx = -1; dx <= 1; ++dx) {
                                const index_t jx = ix + dx, jy = iy + dy, jz = iz + dz;
                                if (jx < 0 || jy < 0 || jz < 0 || jx >= nx || jy >= ny || jz >= nz) continue;
                                const index_t col = (jz * ny + jy) * nx + jx;
                                e.push_back({m, col, col == m ? diag : off});
                            }
                }
        *out = new CsrMatrix(CsrMatrix::from_triplets(n, n, std::move(e)));
    });
}
void ref_csr_free(void *m) { delete static_cast<CsrMatrix *>(m); }
// read_matrix_market / write_matrix_market (inc/mm_io.hpp)
int ref_read_mm(const char *path, void **out) {
    return guard([&] { *out = new CsrMatrix(read_matrix_market(path)); });
}
int ref_write_mm(void *m, const char *path) {
    return guard([&] { write_matrix_market(*static_cast<CsrMatrix *>(m), std::string(path)); });
}
void ref_csr_info(void *m, int32_t *nrows, int32_t *ncols, int64_t *nnz) {
    auto *A = static_cast<CsrMatrix *>(m);
    *nrows = A->nrows();
    *ncols = A->ncols();
    *nnz = A->nnz();
}
void ref_csr_copy(void *m, int32_t *rp, int32_t *ci, double *v) {
    auto *A = static_cast<CsrMatrix *>(m);
    std::memcpy(rp, A->row_ptr().data(), sizeof(int32_t) * A->row_ptr().size());
    std::memcpy(ci, A->col_idx().data(), sizeof(int32_t) * A->col_idx().size());
    std::memcpy(v, A->values().data(), sizeof(double) * A->values().size());
}

// ---- L1 kernels -----------------------------------------------------------
int ref_spmv(void *m, const double *x, double *y) {
    return guard([&] {
        auto *A = static_cast<CsrMatrix *>(m);
        DenseVector out;
        spmv(*A, vec(x, A->ncols()), out);
        std::memcpy(y, out.data(), sizeof(double) * out.size());
    });
}
int ref_spmv_transpose(void *m, const double *x, double *y) {
    return guard([&] {
        auto *A = static_cast<CsrMatrix *>(m);
        const DenseVector out = spmv_transpose(*A, vec(x, A->nrows()));
        std::memcpy(y, out.data(), sizeof(double) * out.size());
    });
}
int ref_residual(void *m, const double *x, const double *f, double *r) {
    return guard([&] {
        auto *A = static_cast<CsrMatrix *>(m);
        const DenseVector out = residual(*A, vec(x, A->ncols()), vec(f, A->nrows()));
        std::memcpy(r, out.data(), sizeof(double) * out.size());
    });
}
int ref_smooth(void *m, int family, double omega, double *x, const double *f, int sweeps) {
    return guard([&] {
        auto *A = static_cast<CsrMatrix *>(m);
        const CycleParams cp = make_cp(family, omega, 0, 0);
        DenseVector xv = vec(x, A->nrows());
        smooth_in_place(cp.smoother, *A, xv, vec(f, A->nrows()), sweeps);
        std::memcpy(x, xv.data(), sizeof(double) * xv.size());
    });
}

// ---- setup ----------------------------------------------------------------
int ref_node_hem(void *m, int32_t *fine_to_coarse, int32_t *n_coarse) {
    return guard([&] {
        const Aggregation agg = coarsen_node_hem(*static_cast<CsrMatrix *>(m));
        std::memcpy(fine_to_coarse, agg.fine_to_coarse.data(),
                    sizeof(int32_t) * agg.fine_to_coarse.size());
        *n_coarse = agg.n_coarse;
    });
}
int ref_galerkin(void *m, const int32_t *fine_to_coarse, int32_t n_coarse, void **out) {
    return guard([&] {
        auto *A = static_cast<CsrMatrix *>(m);
        Aggregation agg{std::vector<index_t>(fine_to_coarse, fine_to_coarse + A->nrows()),
                        n_coarse};
        *out = new CsrMatrix(galerkin_product(*A, agg));
    });
}

int ref_hier_new(void *m, int coarsening, int coarse_target, int max_levels,
                 int coarse_solver, void **out) {
    return guard([&] {
        SolverConfig cfg;
        cfg.coarsening = coarsening == 0 ? CoarseningKind::node_hem : CoarseningKind::edge_hem;
        cfg.coarse_target = coarse_target;
        cfg.max_levels = max_levels;
        cfg.coarse_solver = coarse_solver == 0 ? CoarseSolverKind::direct : CoarseSolverKind::cg;
        auto *rh = new RefHier;
        rh->h = std::make_unique<Hierarchy>(*static_cast<CsrMatrix *>(m), cfg);
        *out = rh;
    });
}
void ref_hier_free(void *h) { delete static_cast<RefHier *>(h); }
int ref_hier_nlevels(void *h) { return static_cast<int>(static_cast<RefHier *>(h)->h->nlevels()); }
int ref_hier_stalled(void *h) { return static_cast<RefHier *>(h)->h->coarsening_stalled() ? 1 : 0; }
void ref_hier_level_info(void *h, int k, int32_t *n, int64_t *nnz, int32_t *n_coarse) {
    const Level &L = static_cast<RefHier *>(h)->h->level(static_cast<std::size_t>(k));
    *n = L.A.nrows();
    *nnz = L.A.nnz();
    *n_coarse = L.agg ? L.agg->n_coarse : -1;
}
void ref_hier_level_copy(void *h, int k, int32_t *rp, int32_t *ci, double *v, int32_t *agg) {
    const Level &L = static_cast<RefHier *>(h)->h->level(static_cast<std::size_t>(k));
    std::memcpy(rp, L.A.row_ptr().data(), sizeof(int32_t) * L.A.row_ptr().size());
    std::memcpy(ci, L.A.col_idx().data(), sizeof(int32_t) * L.A.col_idx().size());
    std::memcpy(v, L.A.values().data(), sizeof(double) * L.A.values().size());
    if (agg && L.agg)
        std::memcpy(agg, L.agg->fine_to_coarse.data(), sizeof(int32_t) * L.agg->fine_to_coarse.size());
}
void *ref_hier_level_matrix(void *h, int k) {
    return const_cast<CsrMatrix *>(&static_cast<RefHier *>(h)->h->level(static_cast<std::size_t>(k)).A);
}
void *ref_hier_level_P(void *h, int k) {
    const Level &L = static_cast<RefHier *>(h)->h->level(static_cast<std::size_t>(k));
    return L.P_to_coarser ? const_cast<CsrMatrix *>(&*L.P_to_coarser) : nullptr;
}
int ref_coarse_solve(void *h, const double *f, double *x) {
    return guard([&] {
        const Hierarchy &H = *static_cast<RefHier *>(h)->h;
        const DenseVector out = H.factorization()->solve(vec(f, H.coarsest().nrows()));
        std::memcpy(x, out.data(), sizeof(double) * out.size());
    });
}
void ref_coarse_counts(void *h, long *symbolic, long *numeric, long *solves) {
    const CoarseFactorization *F = static_cast<RefHier *>(h)->h->factorization();
    *symbolic = F ? F->symbolic_count() : -1;
    *numeric = F ? F->numeric_count() : -1;
    *solves = F ? F->solve_count() : -1;
}

// ---- analytical memory model (inc/memory_model.hpp) ---------------------------
// scheme 0: CI (level streaming), 1: MI (resident hierarchy); BytesModel{8, 4}
int ref_memory_plan(void *h, int scheme, long long *peak, long long *resident, long long *per_cycle) {
    return guard([&] {
        auto *rh = static_cast<RefHier *>(h);
        const MemoryPlan p = scheme == 0 ? plan_ci(*rh->h, rh->cp) : plan_mi(*rh->h, rh->cp);
        *peak = p.peak_device_bytes;
        *resident = p.resident_setup_bytes;
        *per_cycle = p.per_cycle_transfer_bytes;
    });
}
long long ref_csr_bytes(void *m) { return csr_bytes(*static_cast<CsrMatrix *>(m), BytesModel{}); }

// ---- solve phase ----------------------------------------------------------
void ref_hier_set_cycle(void *h, int family, double omega, int pre, int post) {
    static_cast<RefHier *>(h)->cp = make_cp(family, omega, pre, post);
}
int ref_vcycle(void *h, int k, const double *f, double *x) {
    return guard([&] {
        auto *rh = static_cast<RefHier *>(h);
        const auto n = rh->h->level(static_cast<std::size_t>(k)).A.nrows();
        DenseVector xv = vec(x, n);
        vcycle_in_place(*rh->h, static_cast<std::size_t>(k), vec(f, n), xv, rh->cp);
        std::memcpy(x, xv.data(), sizeof(double) * xv.size());
    });
}

static void fill_report(const SolveResult &res, ref_report *rep) {
    rep->iterations = res.report.iterations;
    rep->termination = static_cast<int>(res.report.termination);
    rep->wall_time = res.report.wall_time;
    rep->true_residual = res.report.true_residual;
    rep->hist_len = static_cast<int>(res.report.residual_history.size());
    const int m = rep->hist_len < rep->hist_cap ? rep->hist_len : rep->hist_cap;
    for (int i = 0; i < m; ++i) {
        if (rep->residual_history) rep->residual_history[i] = res.report.residual_history[i];
        if (rep->time_history) rep->time_history[i] = res.report.time_history[i];
    }
}

// solver: 0 pcg, 1 pbicgstab. h == nullptr -> identity preconditioner on A.
int ref_krylov(int solver, void *A, void *h, const double *b, double *x, double tol,
               int max_iters, ref_report *rep) {
    return guard([&] {
        auto *M = static_cast<CsrMatrix *>(A);
        Preconditioner P = h ? make_amg_preconditioner(*static_cast<RefHier *>(h)->h,
                                                       static_cast<RefHier *>(h)->cp)
                             : Preconditioner::identity();
        const DenseVector bv = vec(b, M->nrows());
        const SolveResult res = solver == 0 ? pcg(*M, bv, P, tol, max_iters)
                                            : pbicgstab(*M, bv, P, tol, max_iters);
        std::memcpy(x, res.x.data(), sizeof(double) * res.x.size());
        fill_report(res, rep);
    });
}
int ref_amg_solve(void *h, const double *b, double *x, double tol, int max_cycles,
                  ref_report *rep) {
    return guard([&] {
        auto *rh = static_cast<RefHier *>(h);
        const SolveResult res = amg_solve(*rh->h, vec(b, rh->h->level(0).A.nrows()), tol,
                                          max_cycles, rh->cp);
        std::memcpy(x, res.x.data(), sizeof(double) * res.x.size());
        fill_report(res, rep);
    });
}

} // extern "C"
