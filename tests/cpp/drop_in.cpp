// Drop-in check: reference-style C++ calls against sparsh_b200.hpp (the same
// statements a sparsh caller writes, namespace swapped). Prints one JSON line.
#include <cmath>
#include <cstdio>
#include <vector>

#include "sparsh_b200.hpp"

namespace sb = sparsh_b200;

static sb::CsrMatrix poisson3d(int n) {
    const sb_csr *none = nullptr;
    (void)none;
    sb_csr m{};
    const double off[6] = {-1, -1, -1, -1, -1, -1};
    sb::detail::check(sb_gen_stencil7(n, n, n, 6.0, off, &m));
    const int64_t nnz = m.row_ptr32[m.nrows];
    sb::CsrMatrix A(static_cast<int>(m.nrows), static_cast<int>(m.ncols),
                    std::vector<int>(m.row_ptr32, m.row_ptr32 + m.nrows + 1),
                    std::vector<int>(m.col_idx, m.col_idx + nnz), std::vector<double>(m.values, m.values + nnz));
    sb_free_csr(&m);
    return A;
}

int main() {
    const sb::CsrMatrix A = poisson3d(32);
    sb::SolverConfig cfg;
    cfg.smoother = sb::SmootherKind::weighted_jacobi();
    cfg.max_levels = 40;
    const sb::Hierarchy h(A, cfg);
    const sb::DenseVector b(static_cast<std::size_t>(A.nrows()), 1.0);
    double nb = 0;
    for (double v : b) nb += v * v;
    const double tol = 1e-8 * std::sqrt(nb);
    const auto res = sb::pcg(A, b, sb::make_amg_preconditioner(h, sb::CycleParams::from(cfg)), tol, 200);
    const auto plain = sb::cg(A, b, tol, 2000);
    const auto amg = sb::amg_solve(h, b, tol, 200, sb::CycleParams::from(cfg));
    bool threw = false;
    try {
        sb::pcg(A, b, sb::make_amg_preconditioner(h, sb::CycleParams{}), tol, 10);  // GS default
    } catch (const std::invalid_argument &) {
        threw = true;
    }
    // B200 placement options: hybrid coarse levels on the host + GPU Galerkin products
    const sb::Hierarchy hh(A, cfg, sb::DeviceOptions{0, 4, true});
    const auto rh = sb::pcg(A, b, sb::make_amg_preconditioner(hh, sb::CycleParams::from(cfg)), tol, 200);
    const bool hybrid_same = rh.report.iterations == res.report.iterations && rh.x == res.x && hh.host_bytes() > 0;
    std::printf("{\"levels\": %zu, \"pcg_iters\": %d, \"pcg_converged\": %d, \"cg_iters\": %d, "
                "\"amg_iters\": %d, \"true_residual\": %.3e, \"gs_rejected\": %d, \"hybrid_same\": %d}\n",
                h.nlevels(), res.report.iterations, res.report.converged() ? 1 : 0, plain.report.iterations,
                amg.report.iterations, res.report.true_residual, threw ? 1 : 0, hybrid_same ? 1 : 0);
    return res.report.converged() && threw ? 0 : 1;
}
