"""Hybrid placement (north star (a); paper's MI scheme): the
matrix storage of the coarse levels stays in pinned host memory and the same
device kernels read it over the host link. Results are bit-identical to the
fully device-resident hierarchy; device-resident bytes shrink accordingly."""
import numpy as np
import pytest

from helpers import rel

pytestmark = pytest.mark.gpu


def _cfg(sp):
    return sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)


@pytest.mark.parametrize("mk", [lambda sp: sp.poisson3d(32), lambda sp: sp.convdiff3d(20, 18, 17, 1.0, 100.0, 1.0, 1.0)])
def test_hybrid_vcycle_and_pcg_bitwise(sp, mk, monkeypatch):
    monkeypatch.setenv("SB_TAIL_ROWS", "0")  # same kernel sequence on both sides
    A = mk(sp)
    cfg = _cfg(sp)
    cp = sp.CycleParams.from_config(cfg)
    hd = sp.Hierarchy(A, cfg)
    L = hd.nlevels()
    f = sp.rhs_random(A.nrows(), 7)
    x_dev = sp.vcycle(hd, 0, f, np.zeros(A.nrows()), cp)
    for hf in sorted({L - 1, L // 2, 1}):
        hh = sp.Hierarchy(A, cfg, host_levels_from=hf)
        x_h = sp.vcycle(hh, 0, f, np.zeros(A.nrows()), cp)
        assert np.array_equal(x_h, x_dev), hf
        assert hh.host_bytes() > 0 and hh.device_bytes() < hd.device_bytes()
    b = sp.rhs_ones(A.nrows())
    tol = 1e-8 * np.linalg.norm(b)
    solver = sp.pcg if A.nrows() == 32 ** 3 else sp.pbicgstab
    r_d = solver(A, b, sp.make_amg_preconditioner(hd, cp), tol, 200)
    hh = sp.Hierarchy(A, cfg, host_levels_from=L // 2)
    r_h = solver(A, b, sp.make_amg_preconditioner(hh, cp), tol, 200)
    assert r_h.report.iterations == r_d.report.iterations
    assert np.array_equal(r_h.x, r_d.x)


def test_hybrid_everything_on_host(sp, monkeypatch):
    # every level's matrix on the host (the device keeps only vectors)
    A = sp.poisson2d(64, 64)
    cfg = _cfg(sp)
    hh = sp.Hierarchy(A, cfg, host_levels_from=0)
    hd = sp.Hierarchy(A, cfg)
    b = sp.rhs_ones(A.nrows())
    tol = 1e-8 * np.linalg.norm(b)
    cp = sp.CycleParams.from_config(cfg)
    r_h = sp.pcg(A, b, sp.make_amg_preconditioner(hh, cp), tol, 200)
    r_d = sp.pcg(A, b, sp.make_amg_preconditioner(hd, cp), tol, 200)
    assert r_h.report.converged() and r_h.report.iterations == r_d.report.iterations
    assert rel(r_h.x, r_d.x) < 1e-14
    assert hh.device_bytes() < hd.device_bytes() / 2
