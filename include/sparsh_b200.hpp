// sparsh_b200.hpp — header-only C++20 drop-in for the reference's solve-phase
// API (namespace sparsh, /root/reference/proj/include/sparsh), implemented over
// the C ABI in sparsh_b200.h. A caller of
//
//     sparsh::Hierarchy h(A, cfg);
//     auto res = sparsh::pcg(A, b, sparsh::make_amg_preconditioner(h, p), tol, it);
//
// switches by changing the namespace to sparsh_b200 (and linking
// libsparsh_b200.so). Semantics follow the reference: std::invalid_argument
// for argument / configuration errors, std::runtime_error for numerical
// failure (amg_solve divergence, singular coarse pivot), Krylov outcomes via
// Termination. Deviations (documented in INTEGRATION.md):
//   * the smoother must be weighted Jacobi (Gauss-Seidel is rejected, not emulated);
//   * Preconditioner is the device AMG V-cycle or the identity — an arbitrary
//     host std::function would be a CPU fallback and is not accepted;
//   * one Hierarchy serves one solve at a time (device workspaces are mutable).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sparsh_b200.h"

namespace sparsh_b200 {

using index_t = std::int32_t;        // inc/csr.hpp:22
using DenseVector = std::vector<double>;  // inc/csr.hpp:25

namespace detail {
inline void check(int rc) {
    if (rc == SB_OK) return;
    const std::string msg = sb_last_error();
    if (rc == SB_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
} // namespace detail

// inc/csr.hpp:44-169 (host storage; validated by the library on use)
class CsrMatrix {
public:
    CsrMatrix() = default;
    CsrMatrix(index_t nrows, index_t ncols, std::vector<index_t> row_ptr, std::vector<index_t> col_idx,
              std::vector<double> values)
        : nrows_(nrows), ncols_(ncols), row_ptr_(std::move(row_ptr)), col_idx_(std::move(col_idx)),
          values_(std::move(values)) {
        if (row_ptr_.size() != static_cast<std::size_t>(nrows_) + 1)
            throw std::invalid_argument("CsrMatrix: row_ptr length mismatch");
    }
    index_t nrows() const { return nrows_; }
    index_t ncols() const { return ncols_; }
    index_t nnz() const { return static_cast<index_t>(col_idx_.size()); }
    bool is_square() const { return nrows_ == ncols_; }
    const std::vector<index_t> &row_ptr() const { return row_ptr_; }
    const std::vector<index_t> &col_idx() const { return col_idx_; }
    const std::vector<double> &values() const { return values_; }
    sb_csr abi() const {
        return sb_csr{nrows_, ncols_, row_ptr_.data(), nullptr, col_idx_.data(), values_.data()};
    }
    friend bool operator==(const CsrMatrix &, const CsrMatrix &) = default;

private:
    index_t nrows_ = 0, ncols_ = 0;
    std::vector<index_t> row_ptr_{0};
    std::vector<index_t> col_idx_;
    std::vector<double> values_;
};

// inc/smoother.hpp:22-49
struct SmootherKind {
    enum class Family { weighted_jacobi, gauss_seidel_forward, gauss_seidel_backward, gauss_seidel_symmetric };
    Family family = Family::gauss_seidel_symmetric;
    double omega = 2.0 / 3.0;
    static SmootherKind weighted_jacobi(double omega = 2.0 / 3.0) {
        if (!(omega > 0.0) || omega > 1.0)
            throw std::invalid_argument("SmootherKind: Jacobi weight " + std::to_string(omega) + " outside (0, 1]");
        return {Family::weighted_jacobi, omega};
    }
    static SmootherKind gauss_seidel_symmetric() { return {Family::gauss_seidel_symmetric, 2.0 / 3.0}; }
};

enum class CoarseningKind { node_hem, edge_hem };
enum class CoarseSolverKind { direct, cg };

// inc/config.hpp:81-105
struct SolverConfig {
    CoarseningKind coarsening = CoarseningKind::node_hem;
    SmootherKind smoother = SmootherKind::gauss_seidel_symmetric();
    int pre_sweeps = 6;
    int post_sweeps = 6;
    index_t coarse_target = 500;
    int max_levels = 10;
    double tol = 1e-8;
    int max_iters = 1000;
    CoarseSolverKind coarse_solver = CoarseSolverKind::direct;
};

// inc/cycle.hpp:24-32
struct CycleParams {
    int pre_sweeps = 6;
    int post_sweeps = 6;
    SmootherKind smoother = SmootherKind::gauss_seidel_symmetric();
    static CycleParams from(const SolverConfig &c) { return {c.pre_sweeps, c.post_sweeps, c.smoother}; }
    sb_cycle abi() const {
        return sb_cycle{pre_sweeps, post_sweeps, static_cast<int>(smoother.family), smoother.omega};
    }
};

// inc/convergence.hpp:15-48
enum class Termination { converged, max_iters, breakdown, diverged };
struct ConvergenceReport {
    std::vector<double> residual_history;
    std::vector<double> time_history;
    int iterations = 0;
    Termination termination = Termination::max_iters;
    double wall_time = 0.0;
    double true_residual = 0.0;
    bool converged() const { return termination == Termination::converged; }
};
struct SolveResult {
    DenseVector x;
    ConvergenceReport report;
};

// B200 placement options (no reference counterpart): device ordinal, hybrid
// placement of the coarse levels' matrices in host memory (paper's MI scheme),
// Galerkin products on the GPU (bit-identical to the host / reference).
struct DeviceOptions {
    int device = 0;
    int64_t host_levels_from = -1;  // -1: every level device-resident
    bool galerkin_gpu = false;
};

// inc/hierarchy.hpp:49-93: host setup (bit-exact) + device-resident levels.
class Hierarchy {
public:
    Hierarchy(const CsrMatrix &A, const SolverConfig &cfg, int device = 0)
        : Hierarchy(A, cfg, DeviceOptions{device, -1, false}) {}
    Hierarchy(const CsrMatrix &A, const SolverConfig &cfg, const DeviceOptions &d) : Hierarchy() {
        if (!A.is_square()) throw std::invalid_argument("Hierarchy: matrix must be square");
        const sb_csr a = A.abi();
        const sb_setup_opts o{cfg.coarsening == CoarseningKind::node_hem ? 0 : 1, cfg.coarse_target,
                              cfg.max_levels, cfg.coarse_solver == CoarseSolverKind::direct ? 0 : 1, 0,
                              d.galerkin_gpu ? 1 : 0, d.device};
        sb_hier h = nullptr;
        detail::check(sb_setup(&a, &o, &h));
        hier_.reset(h);
        init_device(d.device, d.host_levels_from);
    }
    // Adopt levels built elsewhere (e.g. a reference sparsh::Hierarchy):
    // levels[k] plus fine_to_coarse[k] for k < nlevels-1.
    Hierarchy(const std::vector<CsrMatrix> &levels, const std::vector<std::vector<index_t>> &aggs,
              int device = 0)
        : Hierarchy() {
        std::vector<sb_csr> ls;
        std::vector<const int32_t *> ag;
        if (levels.empty() || aggs.size() + 1 != levels.size())
            throw std::invalid_argument("Hierarchy: need one aggregation per level but the coarsest");
        for (const auto &m : levels) ls.push_back(m.abi());
        for (std::size_t k = 0; k < aggs.size(); ++k) {
            if (static_cast<std::int64_t>(aggs[k].size()) != levels[k].nrows())
                throw std::invalid_argument("Hierarchy: aggregation " + std::to_string(k) +
                                            " does not cover level " + std::to_string(k));
            ag.push_back(aggs[k].data());
        }
        sb_hier h = nullptr;
        detail::check(sb_hier_from_levels(static_cast<int>(ls.size()), ls.data(), ag.data(), &h));
        hier_.reset(h);
        init_device(device);
    }
    // Single-level device context for matrix-only solves (cg / bicgstab).
    static Hierarchy plain(const CsrMatrix &A, int device = 0) {
        Hierarchy H;
        const sb_csr a = A.abi();
        const sb_setup_opts o{0, 1, 1, -1, 0, 0, 0};
        sb_hier h = nullptr;
        detail::check(sb_setup(&a, &o, &h));
        H.hier_.reset(h);
        H.init_device(device);
        return H;
    }
    std::size_t nlevels() const { return static_cast<std::size_t>(sb_hier_nlevels(hier_.get())); }
    bool coarsening_stalled() const { return sb_hier_stalled(hier_.get()) != 0; }
    sb_ctx ctx() const { return ctx_.get(); }
    int64_t device_bytes() const { return sb_device_bytes(ctx_.get()); }
    int64_t host_bytes() const { return sb_host_bytes(ctx_.get()); }

private:
    Hierarchy() : hier_(nullptr, &sb_hier_free), ctx_(nullptr, &sb_destroy) {}
    void init_device(int device, int64_t host_levels_from = -1) {
        const sb_device_opts o{device, 1, host_levels_from, 0};
        sb_ctx c = nullptr;
        detail::check(sb_create(hier_.get(), &o, &c));
        ctx_.reset(c);
    }
    std::unique_ptr<sb_hier_s, void (*)(sb_hier)> hier_;
    std::unique_ptr<sb_ctx_s, void (*)(sb_ctx)> ctx_;
};

// inc/krylov.hpp:30-36 + inc/cycle.hpp:137-145
struct Preconditioner {
    const Hierarchy *h = nullptr;  // null: identity
    CycleParams params;
    static Preconditioner identity() { return {}; }
};

inline Preconditioner make_amg_preconditioner(const Hierarchy &h, CycleParams p = {}) { return {&h, p}; }

namespace detail {
inline SolveResult run(int (*fn)(sb_ctx, const sb_cycle *, const double *, double *, double, int, sb_report *),
                       sb_ctx ctx, const sb_cycle *cp, const DenseVector &b, double tol, int max_iters) {
    SolveResult out;
    out.x.assign(b.size(), 0.0);
    const int cap = (max_iters > 0 ? max_iters : 0) + 2;
    out.report.residual_history.assign(static_cast<std::size_t>(cap), 0.0);
    out.report.time_history.assign(static_cast<std::size_t>(cap), 0.0);
    sb_report r{0, 0, 0.0, 0.0, 0, cap, out.report.residual_history.data(), out.report.time_history.data()};
    const int rc = fn(ctx, cp, b.data(), out.x.data(), tol, max_iters, &r);
    check(rc);
    out.report.residual_history.resize(static_cast<std::size_t>(std::min(r.hist_len, cap)));
    out.report.time_history.resize(out.report.residual_history.size());
    out.report.iterations = r.iterations;
    out.report.termination = static_cast<Termination>(r.termination);
    out.report.wall_time = r.wall_time;
    out.report.true_residual = r.true_residual;
    return out;
}

inline SolveResult krylov(bool bicg, const Hierarchy &h, const DenseVector &b, const Preconditioner &M,
                          double tol, int max_iters) {
    const sb_cycle cp = M.params.abi();
    return run(bicg ? &sb_pbicgstab : &sb_pcg, h.ctx(), M.h ? &cp : nullptr, b, tol, max_iters);
}
} // namespace detail

// pcg / pbicgstab (inc/krylov.hpp:65,126). The matrix is the hierarchy's
// level 0 (the preconditioner carries it); `A` is accepted for signature
// parity and must be that matrix.
inline SolveResult pcg(const Hierarchy &h, const DenseVector &b, const Preconditioner &M, double tol,
                       int max_iters) {
    return detail::krylov(false, h, b, M, tol, max_iters);
}
inline SolveResult pbicgstab(const Hierarchy &h, const DenseVector &b, const Preconditioner &M, double tol,
                             int max_iters) {
    return detail::krylov(true, h, b, M, tol, max_iters);
}

// Reference signatures: pcg(A, b, M, tol, max_iters). With an AMG
// preconditioner A must be the hierarchy's level-0 matrix; with the identity a
// single-level device context is built for A.
inline SolveResult pcg(const CsrMatrix &A, const DenseVector &b, const Preconditioner &M, double tol,
                       int max_iters) {
    if (b.size() != static_cast<std::size_t>(A.nrows()))
        throw std::invalid_argument("pcg: rhs length " + std::to_string(b.size()) +
                                    " does not match dimension " + std::to_string(A.nrows()));
    if (M.h) return pcg(*M.h, b, M, tol, max_iters);
    const Hierarchy p = Hierarchy::plain(A);
    return pcg(p, b, M, tol, max_iters);
}
inline SolveResult pbicgstab(const CsrMatrix &A, const DenseVector &b, const Preconditioner &M, double tol,
                             int max_iters) {
    if (b.size() != static_cast<std::size_t>(A.nrows()))
        throw std::invalid_argument("pbicgstab: rhs length " + std::to_string(b.size()) +
                                    " does not match dimension " + std::to_string(A.nrows()));
    if (M.h) return pbicgstab(*M.h, b, M, tol, max_iters);
    const Hierarchy p = Hierarchy::plain(A);
    return pbicgstab(p, b, M, tol, max_iters);
}
inline SolveResult cg(const CsrMatrix &A, const DenseVector &b, double tol, int max_iters) {
    return pcg(A, b, Preconditioner::identity(), tol, max_iters);
}
inline SolveResult bicgstab(const CsrMatrix &A, const DenseVector &b, double tol, int max_iters) {
    return pbicgstab(A, b, Preconditioner::identity(), tol, max_iters);
}

// amg_solve (inc/cycle.hpp:91-130): throws std::runtime_error("...diverged...").
inline SolveResult amg_solve(const Hierarchy &h, const DenseVector &b, double tol, int max_cycles,
                             const CycleParams &p = {}) {
    const sb_cycle cp = p.abi();
    return detail::run(&sb_amg_solve, h.ctx(), &cp, b, tol, max_cycles);
}

// vcycle_in_place (inc/cycle.hpp:53-75)
inline void vcycle_in_place(const Hierarchy &h, std::size_t k, const DenseVector &f, DenseVector &x,
                            const CycleParams &p) {
    const sb_cycle cp = p.abi();
    detail::check(sb_vcycle(h.ctx(), &cp, static_cast<int>(k), f.data(), x.data()));
}

} // namespace sparsh_b200
