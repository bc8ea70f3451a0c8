// INTEGRATION.md §2, verbatim in spirit: the REFERENCE builds the hierarchy
// (sparsh::Hierarchy, inc/hierarchy.hpp:51), the device adopts its levels
// through sb_hier_from_levels and runs the solve through sb_pcg. The same
// program also runs the reference's own pcg with its AMG preconditioner
// (inc/krylov.hpp:65, inc/cycle.hpp:137) and the product's own setup
// (sb_setup) on the same matrix. Prints one JSON line for
// tests/test_gpu_integration.py.
//
// Test infrastructure: compiled by oracle/Makefile (target `ref`) against the
// reference headers where they lie, linked to libsparsh_b200.so; the binary
// lands in oracle/_ref/ and travels to the GPU box with it.
#include <cmath>
#include <string>
#include <cstdio>
#include <vector>

#include "sparsh/sparsh.hpp"
#include "sparsh_b200.h"

static double rel(const std::vector<double> &a, const std::vector<double> &b) {
    double d = 0, n = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        d += (a[i] - b[i]) * (a[i] - b[i]);
        n += b[i] * b[i];
    }
    return std::sqrt(d / n);
}

static int run_pcg(sb_hier dh, const std::vector<double> &b, double tol, int max_it, std::vector<double> &x,
                   sb_report &rep, std::vector<double> &hist, std::vector<double> &th) {
    sb_ctx ctx = nullptr;
    sb_device_opts o{0, 1, -1, 0};
    if (sb_create(dh, &o, &ctx) != SB_OK) return -1;
    sb_cycle cp{6, 6, SB_SMOOTHER_JACOBI, 2.0 / 3.0};
    x.assign(b.size(), 0.0);
    hist.assign(max_it + 2, 0.0);
    th.assign(max_it + 2, 0.0);
    rep = sb_report{0, 0, 0, 0, 0, max_it + 2, hist.data(), th.data()};
    const int rc = sb_pcg(ctx, &cp, b.data(), x.data(), tol, max_it, &rep);
    sb_destroy(ctx);
    return rc;
}

int main() {
    // 2D 5-point Poisson 128^2 (inc/problems.hpp:60), the reference's own generator
    const sparsh::CsrMatrix A = sparsh::poisson2d(128, 128);
    sparsh::SolverConfig cfg;
    cfg.smoother = sparsh::SmootherKind::weighted_jacobi();
    cfg.max_levels = 40;
    const sparsh::Hierarchy h(A, cfg);  // reference setup (hierarchy.hpp:51)

    std::vector<sb_csr> lv;
    std::vector<const int32_t *> agg;
    for (const auto &L : h.levels()) {
        lv.push_back({L.A.nrows(), L.A.ncols(), L.A.row_ptr().data(), nullptr, L.A.col_idx().data(),
                      L.A.values().data()});  // zero-copy views
        if (L.agg) agg.push_back(L.agg->fine_to_coarse.data());
    }
    sb_hier dh = nullptr;
    if (sb_hier_from_levels((int)lv.size(), lv.data(), agg.data(), &dh) != SB_OK) {
        std::fprintf(stderr, "sb_hier_from_levels: %s\n", sb_last_error());
        return 1;
    }
    // the product's own setup of the same matrix
    sb_hier sh = nullptr;
    sb_csr a0{A.nrows(), A.ncols(), A.row_ptr().data(), nullptr, A.col_idx().data(), A.values().data()};
    sb_setup_opts so{0, 500, 40, 0, 0, 0, 0};
    if (sb_setup(&a0, &so, &sh) != SB_OK) return 2;

    const sparsh::DenseVector b = sparsh::rhs_ones(A.nrows());
    const double tol = 1e-8 * sparsh::norm2(b);
    const int max_it = 500;
    std::vector<double> xa, xs, ha, hs, ta, ts;
    sb_report ra{}, rs{};
    if (run_pcg(dh, b, tol, max_it, xa, ra, ha, ta) != SB_OK) {
        std::fprintf(stderr, "sb_pcg (adopted): %s\n", sb_last_error());
        return 3;
    }
    if (run_pcg(sh, b, tol, max_it, xs, rs, hs, ts) != SB_OK) return 4;
    bool bitwise = ra.iterations == rs.iterations;
    for (size_t i = 0; bitwise && i < xa.size(); ++i) bitwise = xa[i] == xs[i];

    // the reference's own solve with its own preconditioner
    sparsh::CycleParams cp;
    cp.smoother = sparsh::SmootherKind::weighted_jacobi();
    const auto M = sparsh::make_amg_preconditioner(h, cp);
    const sparsh::SolveResult r = sparsh::pcg(A, b, M, tol, max_it);
    // equal iteration count: the solutions must agree to 1e-10
    std::vector<double> xk, hk, tk;
    sb_report rk{};
    if (run_pcg(dh, b, 1e-300, r.report.iterations, xk, rk, hk, tk) != SB_OK) return 5;
    const double err = rel(xk, r.x);

    // a malformed adoption must be rejected with the reference's message
    std::vector<int32_t> bad(agg[0], agg[0] + lv[0].nrows);
    bad[2] = bad[0];  // aggregate agg[0] now holds 3 fine nodes
    std::vector<const int32_t *> agg_bad(agg);
    agg_bad[0] = bad.data();
    sb_hier dbad = nullptr;
    const int rc_bad = sb_hier_from_levels((int)lv.size(), lv.data(), agg_bad.data(), &dbad);
    const bool msg_ok = rc_bad == SB_EINVAL && std::string(sb_last_error()).find("Aggregation: coarse node") == 0;

    std::printf("{\"levels\": %zu, \"adopted_iters\": %d, \"setup_iters\": %d, \"ref_iters\": %d, "
                "\"adopted_converged\": %d, \"adopted_eq_setup_bitwise\": %d, \"rel_err_equal_iters\": %.3e, "
                "\"bad_agg_rejected\": %d}\n",
                h.nlevels(), ra.iterations, rs.iterations, r.report.iterations, ra.termination == 0 ? 1 : 0,
                bitwise ? 1 : 0, err, msg_ok ? 1 : 0);
    sb_hier_free(dh);
    sb_hier_free(sh);
    return 0;
}
