"""Parity at the BASELINE configurations (SURVEY.md §8c protocol, north_star bar).

Two kinds of evidence, both against the REFERENCE's own code (oracle/_ref):

* golden fixtures (tests/golden/config_<name>.npz, written by
  tests/golden/make_config_fixtures.py, which ran the reference on the full
  systems): C1 2D 1024^2, C2 128^3, C3 aniso 256^3, C4 convection-diffusion
  256^3 (BiCGStab), the north-star target T256 (7-pt Poisson 256^3) and the
  27-point 128^3 proxy of C5 (P27_128);
* live runs of the reference on this host for C1 and C2 (full solution vectors).

Asserted per configuration:
  - setup bit-exact: every level's n, nnz and CRC32 of row_ptr / col_idx /
    values / aggregates equal the reference's (hierarchy.hpp:51-76);
  - to-tolerance solve: iterations within +-1, converged, final recurrence
    residual < tol, true relative residual <= 1e-8 (+ rounding slack);
  - equal iteration count (tol = 1e-300, max_iters = k_ref): solution within
    1e-10 relative L2 (on the fixture's strided sample, plus ||x||, sum x and
    x.g over the full vector), residual histories within 1e-8 relative; the
    to-tolerance solution equals the reference's to-tolerance one (for
    BiCGStab both end in the half-step exit when it fires).
"""
import json
import os
import zlib

import numpy as np
import pytest

from conftest import golden_path
from helpers import rel

pytestmark = pytest.mark.gpu

GEN = {
    "C1": lambda sp: sp.poisson2d(1024, 1024),
    "C2": lambda sp: sp.poisson3d(128),
    "C3": lambda sp: sp.aniso3d(256, 1e-3),
    "C4": lambda sp: sp.convdiff3d(256, 256, 256, 1.0, 100.0, 1.0, 1.0),
    "T256": lambda sp: sp.poisson3d(256),
    "P27_128": lambda sp: sp.poisson3d_27(128),
}
CONFIGS = [c for c in ["C1", "C2", "P27_128", "T256", "C3", "C4"] if os.path.exists(golden_path(f"config_{c}.npz"))]


def _crc(a):
    return int(zlib.crc32(np.ascontiguousarray(a).view(np.uint8)))


def _g(n):
    return np.random.default_rng(20070056).standard_normal(n)


class Case:
    def __init__(self, sp, name):
        z = np.load(golden_path(f"config_{name}.npz"))
        self.meta = json.loads(str(z["meta"]))
        self.x_sample = z["x_sample"]
        self.xe_sample = z["xe_sample"] if "xe_sample" in z.files else z["x_sample"]
        self.hist = z["residual_history"]
        self.name = name
        self.A = GEN[name](sp)
        cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40, coarse_target=500)
        self.h = sp.Hierarchy(self.A, cfg)
        self.cp = sp.CycleParams.from_config(cfg)
        self.M = sp.make_amg_preconditioner(self.h, self.cp)
        self.solve = getattr(sp, self.meta["solver"])
        self.b = sp.rhs_ones(self.A.nrows())


@pytest.fixture(scope="module", params=CONFIGS)
def case(request, sp):
    c = Case(sp, request.param)
    yield c
    del c


def test_config_setup_bitexact(case):
    """Aggregates and every coarse operator equal the reference's, bit for bit."""
    m = case.meta
    assert case.A.nrows() == m["n"] and case.A.nnz() == m["nnz"]
    lv = case.h.levels()
    assert len(lv) == len(m["levels"])
    for k, (L, R) in enumerate(zip(lv, m["levels"])):
        assert (L.A.nrows(), L.A.nnz()) == (R["n"], R["nnz"]), k
        assert _crc(np.asarray(L.A.row_ptr(), dtype=np.int32)) == R["crc_rp"], k
        assert _crc(np.asarray(L.A.col_idx(), dtype=np.int32)) == R["crc_ci"], k
        assert _crc(np.asarray(L.A.values(), dtype=np.float64)) == R["crc_v"], k
        if R["crc_agg"] is not None:
            assert _crc(np.asarray(L.agg.fine_to_coarse, dtype=np.int32)) == R["crc_agg"], k
    case.h._levels = None  # drop the host copies (1.4 GB at 256^3)


def test_config_to_tolerance(case):
    """Iterations within +-1 of the reference, same 1e-8 tolerance reached."""
    m = case.meta
    tol = m["tol"]
    res = case.solve(case.A, case.b, case.M, tol, 1000)
    rep = res.report
    assert rep.converged(), rep.termination
    assert abs(rep.iterations - m["iterations"]) <= 1, (rep.iterations, m["iterations"])
    assert rep.residual_history[-1] < tol
    assert len(rep.residual_history) == rep.iterations + 1
    nb = float(np.linalg.norm(case.b))
    assert rep.true_residual / nb < 1.5e-8, rep.true_residual / nb
    if rep.iterations == m["iterations"]:
        assert abs(rep.true_residual - m["true_residual"]) <= 0.05 * m["true_residual"] + 1e-3 * tol
        # the same exit (incl. BiCGStab's half-step exit, krylov.hpp:167-173): same iterate
        assert rel(res.x[::m["stride"]], case.x_sample) < 1e-10


def test_config_equal_iterations(case):
    """At the reference's iteration count the solutions agree to 1e-10 relative L2."""
    m = case.meta
    k = m["iterations"]
    res = case.solve(case.A, case.b, case.M, 1e-300, k)
    assert res.report.iterations == k
    x = res.x
    pre = "xe_" if "xe_norm2" in m else "x_"
    assert rel(x[::m["stride"]], case.xe_sample) < 1e-10
    assert abs(np.linalg.norm(x) - m[pre + "norm2"]) <= 1e-10 * m[pre + "norm2"]
    assert abs(x @ _g(x.size) - m[pre + "dot_g"]) <= 1e-10 * np.linalg.norm(x) * np.sqrt(x.size)
    assert abs(np.sum(x) - m[pre + "sum"]) <= 1e-10 * np.sum(np.abs(x))
    hist = np.asarray(res.report.residual_history)
    assert hist.size == case.hist.size
    # (a BiCGStab half-step exit records ||s|| last where this run records ||r||)
    m_ = hist.size - 1 if m["solver"] != "pcg" else hist.size
    assert rel(hist[:m_], case.hist[:m_]) < 1e-8


@pytest.mark.parametrize("name,rhs", [("C1", "ones"), ("C2", "ones"), ("C2", "random")])
def test_config_live_vs_reference(sp, ref, name, rhs):
    """Full solution vectors against the reference run here (C1, C2)."""
    A = GEN[name](sp)
    n = A.nrows()
    b = sp.rhs_ones(n) if rhs == "ones" else sp.rhs_random(n, 42)
    tol = 1e-8 * float(np.linalg.norm(b))
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40, coarse_target=500)
    h = sp.Hierarchy(A, cfg)
    M = sp.make_amg_preconditioner(h, sp.CycleParams.from_config(cfg))
    ref.set_threads(os.cpu_count() or 1)
    rh = ref.hierarchy(ref.problem(name), 500, 40)
    o = rh.pcg(b, tol, 1000)
    res = sp.pcg(A, b, M, tol, 1000)
    assert res.report.converged() and o.termination == 0
    assert abs(res.report.iterations - o.iterations) <= 1
    k = o.iterations
    r2 = sp.pcg(A, b, M, 1e-300, k)
    assert rel(r2.x, o.x) < 1e-10
    assert rel(r2.report.residual_history, o.residual_history) < 1e-8
