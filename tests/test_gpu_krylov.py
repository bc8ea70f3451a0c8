"""Krylov drivers on the GPU vs the reference (krylov.hpp, cycle.hpp:91-130).
Contract (BASELINE.json north_star): iterations within +-1, converged residual
below the same tolerance, solutions within 1e-10 relative L2 — compared at the
SAME iteration count (tol = 1e-300, max_iters = k_ref; SURVEY §8c protocol)."""
import glob

import numpy as np
import pytest

from conftest import golden_path
from helpers import from_npz, random_sparse, rel

pytestmark = pytest.mark.gpu


def _cfg(sp, **kw):
    return sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40, **kw)


def _cp(sp):
    return sp.CycleParams.from_config(_cfg(sp))


PROBLEMS = {
    "poisson3d_40": (lambda sp: sp.poisson3d(40), "pcg"),
    "aniso3d_32": (lambda sp: sp.aniso3d(32), "pcg"),
    "poisson2d_128": (lambda sp: sp.poisson2d(128, 128), "pcg"),
    "poisson27_20": (lambda sp: sp.poisson3d_27(20), "pcg"),
    "convdiff3d_24": (lambda sp: sp.convdiff3d(24, 24, 24, 1.0, 100.0, 1.0, 1.0), "pbicgstab"),
    "convdiff2d_64": (lambda sp: sp.convdiff2d(64, 64, 1.0, 100.0, 1.0), "pbicgstab"),
}


@pytest.mark.parametrize("name", sorted(PROBLEMS))
@pytest.mark.parametrize("rhs", ["ones", "random"])
def test_krylov_parity(sp, port, name, rhs):
    mk, solver = PROBLEMS[name]
    A = mk(sp)
    n = A.nrows()
    b = sp.rhs_ones(n) if rhs == "ones" else sp.rhs_random(n, 42)
    tol = 1e-8 * np.linalg.norm(b)
    h = sp.Hierarchy(A, _cfg(sp))
    M = sp.make_amg_preconditioner(h, _cp(sp))
    o = port.hierarchy(A, 500, 40)
    fn = getattr(sp, solver)
    res = fn(A, b, M, tol, 500)
    ref = getattr(o, solver)(b, tol, 500)
    assert res.report.converged() and ref.termination == 0
    assert abs(res.report.iterations - ref.iterations) <= 1
    assert res.report.residual_history[-1] < tol
    assert len(res.report.residual_history) == res.report.iterations + 1
    assert res.report.true_residual < 10 * tol
    assert abs(res.report.residual_history[0] - ref.residual_history[0]) <= 1e-14 * ref.residual_history[0]
    # same iteration count -> solutions agree to 1e-10
    k = ref.iterations
    r2 = fn(A, b, M, 1e-300, k)
    o2 = getattr(o, solver)(b, 1e-300, k)
    assert r2.report.iterations == o2.iterations == k
    assert rel(r2.x, o2.x) < 1e-10
    assert rel(r2.report.residual_history, o2.residual_history) < 1e-8


@pytest.mark.parametrize("path", sorted(p for p in glob.glob(golden_path("*.npz"))
                                        if not p.endswith("example_6x6.npz") and "config_" not in p))
def test_golden_solves(sp, port, path):
    d = np.load(path)
    A = from_npz(sp, d)
    h = sp.Hierarchy(A, _cfg(sp, coarse_target=100))
    assert h.nlevels() == int(d["nlevels"])
    M = sp.make_amg_preconditioner(h, _cp(sp))
    assert rel(sp.vcycle(h, 0, d["b"], np.zeros(A.nrows()), _cp(sp)), d["vcycle"]) < 1e-12
    solver = str(d["solver"])
    res = getattr(sp, solver)(A, d["b"], M, float(d["tol"]), 500)
    assert abs(res.report.iterations - int(d["iters"])) <= 1
    assert res.report.termination == int(d["term"])
    if res.report.iterations == int(d["iters"]):  # same exit point (incl. BiCGStab half step)
        assert rel(res.x, d["x"]) < 1e-10
        assert rel(res.report.residual_history, d["hist"]) < 1e-8
    k = int(d["iters"])
    same = getattr(sp, solver)(A, d["b"], M, 1e-300, k)
    o = port.hierarchy(A, 100, 40)
    assert rel(same.x, getattr(o, solver)(d["b"], 1e-300, k).x) < 1e-10
    amg = sp.amg_solve(h, d["b"], float(d["tol"]), 40, _cp(sp))
    assert abs(amg.report.iterations - int(d["amg_iters"])) <= 1
    assert rel(sp.amg_solve(h, d["b"], 1e-300, int(d["amg_iters"]), _cp(sp)).x, d["amg_x"]) < 1e-10


def test_amg_solve_parity_and_report(sp, port):
    # test_cycle.cpp:102-122
    A = sp.poisson2d(64, 64)
    h = sp.Hierarchy(A, _cfg(sp))
    b = sp.rhs_ones(4096)
    res = sp.amg_solve(h, b, 1e-8, 200, _cp(sp))
    o = port.hierarchy(A, 500, 40).amg_solve(b, 1e-8, 200)
    assert res.report.converged() and abs(res.report.iterations - o.iterations) <= 1
    assert len(res.report.residual_history) == res.report.iterations + 1
    assert len(res.report.time_history) == len(res.report.residual_history)
    assert all(t1 >= t0 for t0, t1 in zip(res.report.time_history, res.report.time_history[1:]))
    assert res.report.residual_history[-1] == res.report.true_residual
    assert np.linalg.norm(sp.residual(A, res.x, b)) < 1e-8
    mx = sp.amg_solve(h, b, 1e-300, 3, _cp(sp))
    assert mx.report.termination == sp.Termination.max_iters and mx.report.iterations == 3
    z = sp.amg_solve(h, np.zeros(4096), 1e-8, 10, _cp(sp))
    assert z.report.iterations == 0 and z.report.converged() and not z.x.any()


def test_amg_divergence_raises(sp):
    # test_cycle.cpp:135-148: [[1,3],[3,1]] diverges -> runtime_error("...diverged...")
    A = sp.CsrMatrix.from_dense([[1.0, 3.0], [3.0, 1.0]])
    h = sp.Hierarchy(A, _cfg(sp, coarse_target=1))
    with pytest.raises(RuntimeError, match="diverged"):
        sp.amg_solve(h, [1.0, -1.0], 1e-8, 50, _cp(sp))


def test_termination_semantics(sp):
    # test_krylov.cpp:14-19, 78-112, 140-147
    r = sp.cg(sp.CsrMatrix.identity(5), sp.rhs_ones(5), 1e-12, 10)
    assert r.report.converged() and r.report.iterations == 1 and np.all(r.x == 1.0)
    A = sp.CsrMatrix.from_triplets(2, 2, [(0, 0, 1.0), (1, 1, -1.0)])
    r = sp.cg(A, [1.0, 1.0], 1e-10, 10)
    assert r.report.termination == sp.Termination.breakdown and r.report.iterations == 0
    r = sp.cg(sp.poisson2d(16, 16), sp.rhs_ones(256), 1e-300, 4)
    assert r.report.termination == sp.Termination.max_iters and r.report.iterations == 4
    assert len(r.report.residual_history) == 5 and len(r.report.time_history) == 5
    r = sp.cg(sp.poisson2d(4, 4), sp.zeros(16), 1e-8, 10)
    assert r.report.converged() and r.report.iterations == 0 and not r.x.any()
    r = sp.bicgstab(sp.CsrMatrix.identity(4), sp.rhs_ones(4), 1e-10, 10)
    assert r.report.converged() and r.report.iterations == 1 and np.all(r.x == 1.0)
    assert r.report.residual_history[-1] == 0.0
    R = sp.CsrMatrix.from_triplets(2, 2, [(0, 1, 1.0), (1, 0, -1.0)])
    assert sp.bicgstab(R, [1.0, 0.0], 1e-10, 10).report.termination == sp.Termination.breakdown


def test_plain_cg_matches_textbook(sp, port):
    # test_krylov.cpp:34-48: pcg(identity) == textbook CG (1e-12 here: tree-order dots)
    A = sp.poisson2d(32, 32)
    b = sp.rhs_ones(1024)
    lib = sp.pcg(A, b, sp.Preconditioner.identity(), 1e-300, 5)
    o = port.hierarchy(A, 500, 40).pcg(b, 1e-300, 5, amg=False)
    assert rel(lib.x, o.x) < 1e-12
    assert rel(lib.report.residual_history, o.residual_history) < 1e-12


def test_bicgstab_unsymmetric(sp, port):
    A = random_sparse(sp, 40, 127, 0.25, False)
    b = np.random.default_rng(0).uniform(-1, 1, 40)
    tol = 1e-9 * np.linalg.norm(b)
    r = sp.bicgstab(A, b, tol, 300)
    o = port.hierarchy(A, 500, 40).pbicgstab(b, tol, 300, amg=False)
    assert r.report.converged() and abs(r.report.iterations - o.iterations) <= 1
    assert np.max(np.abs(r.x - o.x)) < 1e-6


def test_amg_beats_plain_and_determinism(sp):
    A = sp.poisson2d(32, 32)
    b = sp.rhs_ones(1024)
    h = sp.Hierarchy(A, _cfg(sp))
    pre = sp.pcg(A, b, sp.make_amg_preconditioner(h, _cp(sp)), 1e-8, 1000)
    plain = sp.cg(A, b, 1e-8, 1000)
    assert pre.report.converged() and plain.report.converged()
    assert pre.report.iterations < plain.report.iterations
    again = sp.pcg(A, b, sp.make_amg_preconditioner(h, _cp(sp)), 1e-8, 1000)
    assert np.array_equal(pre.x, again.x)
    assert pre.report.residual_history == again.report.residual_history


def test_bad_arguments(sp):
    A = sp.poisson2d(4, 4)
    with pytest.raises(sp.InvalidArgument):
        sp.cg(A, sp.rhs_ones(15), 1e-8, 10)
    with pytest.raises(sp.InvalidArgument):
        sp.cg(A, sp.rhs_ones(16), 0.0, 10)
    with pytest.raises(sp.InvalidArgument):
        sp.bicgstab(A, sp.rhs_ones(16), -1.0, 10)


def test_c2_shape_64cubed(sp, port):
    # 64^3 7-pt PCG: 16 iterations in the survey probe
    A = sp.poisson3d(64)
    b = sp.rhs_ones(A.nrows())
    tol = 1e-8 * np.linalg.norm(b)
    h = sp.Hierarchy(A, _cfg(sp))
    res = sp.pcg(A, b, sp.make_amg_preconditioner(h, _cp(sp)), tol, 100)
    assert res.report.converged() and res.report.iterations == 16
    o = port.hierarchy(A, 500, 40).pcg(b, 1e-300, 16)
    r2 = sp.pcg(A, b, sp.make_amg_preconditioner(h, _cp(sp)), 1e-300, 16)
    assert rel(r2.x, o.x) < 1e-10


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_deferred_x_update_bitwise(graphs):
    """PCG with x += alpha p moved into the p update (k_xpay_x) or the post-loop
    k_x_final: the same operation on the same values, so the solution, the
    iteration count and the residual history equal the in-place update
    (SB_DEFER_X=0) bit for bit -- also for a solve that stops at max_iters and
    for plain CG (no preconditioner)."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import sys, numpy as np; sys.path.insert(0, %r); from paper_2007_00056_b200 import sparsh as sp; "
            "A = sp.poisson3d(40, 36, 30); "
            "cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40); "
            "h = sp.Hierarchy(A, cfg, graphs=%s); cp = sp.CycleParams.from_config(cfg); "
            "b = sp.rhs_random(A.nrows(), 11); M = sp.make_amg_preconditioner(h, cp); "
            "out = []\n"
            "for tol, k in ((1e-8 * np.linalg.norm(b), 200), (1e-14 * np.linalg.norm(b), 5)):\n"
            "    r = sp.pcg(A, b, M, tol, k)\n"
            "    out += [r.x.tobytes().hex(), str(r.report.iterations), np.asarray(r.report.residual_history).tobytes().hex()]\n"
            "r = sp.cg(A, b, 1e-8 * np.linalg.norm(b), 300)\n"
            "out += [r.x.tobytes().hex(), str(r.report.iterations)]\n"
            "sys.stdout.write(' '.join(out))")
    outs = []
    for on in ("1", "0"):
        p = subprocess.run([sys.executable, "-c", code % (ROOT, "True" if graphs == "1" else "False")],
                           env=dict(os.environ, SB_DEFER_X=on), capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(p.stdout.split())
    assert outs[0] and outs[0] == outs[1]
