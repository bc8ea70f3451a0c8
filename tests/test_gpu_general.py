"""General-valued operators (every row distinct: no row patterns, no value
dictionary, irregular node-HEM coarse levels) take the SELL-G / CSR-tile
formats. The V-cycle must stay bit-identical to the reference with the exact
coarse solve (inc/cycle.hpp:53-75), PCG must agree within the contract, and
contexts created later in the process (smaller tiles) must not break an
earlier context's launches (shared-memory function attributes are process-wide)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(sp):
    return sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)


def test_graph_laplacian_vcycle_bitexact(sp, port):
    A = sp.graph_laplacian3d(20, seed=3)
    h = sp.Hierarchy(A, _cfg(sp), device=0, coarse_exact=True)
    o = port.hierarchy(A, 500, 40)
    assert h.nlevels() == o.nlevels()
    f = np.random.default_rng(4).uniform(-1, 1, A.nrows())
    cp = sp.CycleParams.from_config(_cfg(sp))
    got = sp.vcycle(h, 0, f, np.zeros(A.nrows()), cp)
    assert np.array_equal(got, o.vcycle(f, np.zeros(A.nrows())))


def test_graph_laplacian_pcg_matches_oracle(sp, oracle_best):
    A = sp.graph_laplacian3d(24, seed=5)
    b = sp.rhs_ones(A.nrows())
    tol = 1e-8 * float(np.linalg.norm(b))
    h = sp.Hierarchy(A, _cfg(sp), device=0)
    res = sp.pcg(A, b, sp.make_amg_preconditioner(h, sp.CycleParams.from_config(_cfg(sp))), tol, 300)
    ref = oracle_best.hierarchy(A, 500, 40).pcg(b, tol, 300)
    assert res.report.converged()
    assert abs(res.report.iterations - ref.iterations) <= 1
    assert np.linalg.norm(res.x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)


def test_later_context_keeps_earlier_launches_valid(sp):
    # bench.py's sequence: a hierarchy, then a single-level context for a
    # residual check, then more launches on the first context
    A = sp.graph_laplacian3d(48, seed=7)
    cfg = _cfg(sp)
    h = sp.Hierarchy(A, cfg, device=0)
    cp = sp.CycleParams.from_config(cfg)
    f = sp.rhs_ones(A.nrows())
    v1 = sp.vcycle(h, 0, f, np.zeros(A.nrows()), cp)
    for B in (sp.poisson3d(9), sp.graph_laplacian3d(6, seed=1), A):
        sp.residual(B, np.ones(B.nrows()), np.ones(B.nrows()))
    v2 = sp.vcycle(h, 0, f, np.zeros(A.nrows()), cp)
    assert np.array_equal(v1, v2)


def _long_rows(sp, n=3000, seed=11):
    # tridiagonal plus rows of 33..700 entries (hubs, as node-HEM coarse levels
    # of irregular graphs grow them): the CSR-tile kernel's warp-per-row path
    rng = np.random.default_rng(seed)
    ent = {}
    for i in range(n):
        ent[(i, i)] = 10.0 + rng.uniform(0, 1)
        if i:
            ent[(i, i - 1)] = -rng.uniform(0.1, 1)
        if i + 1 < n:
            ent[(i, i + 1)] = -rng.uniform(0.1, 1)
    for r, L in [(5, 33), (6, 64), (300, 129), (301, 700), (302, 40), (1000, 255), (2999, 97)]:
        for c in rng.choice(n, L, replace=False):
            ent[(r, int(c))] = ent.get((r, int(c)), 0.0) - rng.uniform(0.001, 0.01)
    return sp.CsrMatrix.from_triplets(n, n, [(r, c, v) for (r, c), v in ent.items()])


def test_long_rows_warp_path_bitexact(sp, oracle_best):
    A = _long_rows(sp)
    assert np.diff(A.row_ptr()).max() > 600
    x = np.random.default_rng(1).uniform(-1, 1, A.ncols())
    f = np.random.default_rng(2).uniform(-1, 1, A.nrows())
    assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x))
    assert np.array_equal(sp.residual(A, x, f), oracle_best.residual(A, x, f))
    jac = sp.SmootherKind.weighted_jacobi()
    assert np.array_equal(sp.smooth(jac, A, x, f, 3), oracle_best.jacobi(A, 2.0 / 3.0, x, f, 3))


def test_long_rows_vcycle_bitexact(sp, port):
    A = _long_rows(sp, n=6000, seed=12)
    cfg = _cfg(sp)
    h = sp.Hierarchy(A, cfg, device=0, coarse_exact=True)
    o = port.hierarchy(A, 500, 40)
    f = np.random.default_rng(3).uniform(-1, 1, A.nrows())
    got = sp.vcycle(h, 0, f, np.zeros(A.nrows()), sp.CycleParams.from_config(cfg))
    assert np.array_equal(got, o.vcycle(f, np.zeros(A.nrows())))
