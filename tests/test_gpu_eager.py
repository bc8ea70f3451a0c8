"""Eager launch mode (sb_device_opts.use_graphs = 0): the solve drivers emit
the same kernels onto the stream with host-side loop control instead of one
whole-solve graph with conditional nodes. Results must be bit-identical to the
graph path, and the kernels the graph executed (counted from its structure,
sb_last_solve_launches) must equal the kernels the eager run launched."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "pcg_poisson3d_24": (lambda sp: sp.poisson3d(24), "pcg"),
    "pcg_poisson2d_96": (lambda sp: sp.poisson2d(96, 96), "pcg"),
    "bicg_convdiff3d_16": (lambda sp: sp.convdiff3d(16, 16, 16, 1.0, 100.0, 1.0, 1.0), "pbicgstab"),
    "amg_aniso3d_16": (lambda sp: sp.aniso3d(16), "amg_solve"),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("tol_mode", ["converge", "maxit"])
def test_eager_equals_graph(sp, name, tol_mode):
    mk, solver = CASES[name]
    A = mk(sp)
    b = sp.rhs_random(A.nrows(), 42)
    tol = 1e-8 * np.linalg.norm(b) if tol_mode == "converge" else 1e-300
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
    cp = sp.CycleParams.from_config(cfg)
    out = {}
    for graphs in (True, False):
        h = sp.Hierarchy(A, cfg, graphs=graphs)
        if solver == "amg_solve":
            res = sp.amg_solve(h, b, tol, 7 if tol_mode == "maxit" else 200, cp)
        else:
            res = getattr(sp, solver)(A, b, sp.make_amg_preconditioner(h, cp), tol, 5 if tol_mode == "maxit" else 200)
        out[graphs] = (res, h.last_solve_launches())
    (rg, lg), (re, le) = out[True], out[False]
    assert rg.report.iterations == re.report.iterations
    assert rg.report.termination == re.report.termination
    assert np.array_equal(rg.x.view(np.uint64), re.x.view(np.uint64))
    assert rg.report.residual_history == re.report.residual_history
    assert lg == le and le > 0
