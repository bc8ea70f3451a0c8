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


HYB = {
    "poisson3d_32": (lambda sp: sp.poisson3d(32), "pcg"),
    "graph_laplacian_20": (lambda sp: sp.graph_laplacian3d(20, seed=3), "pcg"),
    "convdiff3d_20": (lambda sp: sp.convdiff3d(20, 18, 17, 1.0, 100.0, 1.0, 1.0), "pbicgstab"),
}


@pytest.mark.parametrize("name", sorted(HYB))
def test_hybrid_vs_reference(sp, oracle_best, name):
    """Hybrid placement against the REFERENCE (not the device path): one V-cycle
    within 1e-12, solves with iterations +-1 and, at equal iteration counts,
    solutions within 1e-10, for several host_levels_from."""
    mk, solver = HYB[name]
    A = mk(sp)
    cfg = _cfg(sp)
    cp = sp.CycleParams.from_config(cfg)
    o = oracle_best.hierarchy(A, 500, 40)
    f = sp.rhs_random(A.nrows(), 11)
    v_ref = o.vcycle(f, np.zeros(A.nrows()))
    b = sp.rhs_ones(A.nrows())
    tol = 1e-8 * np.linalg.norm(b)
    ref = getattr(o, solver)(b, tol, 300)
    k = ref.iterations
    ref_k = getattr(o, solver)(b, 1e-300, k)
    L = sp.Hierarchy(A, cfg).nlevels()
    for hf in sorted({1, L // 2, L - 1}):
        hh = sp.Hierarchy(A, cfg, host_levels_from=hf)
        assert rel(sp.vcycle(hh, 0, f, np.zeros(A.nrows()), cp), v_ref) < 1e-12, hf
        M = sp.make_amg_preconditioner(hh, cp)
        r = getattr(sp, solver)(A, b, M, tol, 300)
        assert r.report.converged() and abs(r.report.iterations - k) <= 1, hf
        rk = getattr(sp, solver)(A, b, M, 1e-300, k)
        assert rel(rk.x, ref_k.x) < 1e-10, hf


def test_hybrid_residency_vs_memory_model(sp, ref):
    """Residency of the MI-style placement (every level but the coarsest on the
    device, inc/memory_model.hpp plan_mi) against the reference's byte model:
    the coarsest level's storage is on the host and every other level's on the
    device (sb_level_residency); the device-resident matrices stream no more
    than the model's csr_bytes of the same levels (per level the f64 SELL-G
    slices may pad a little past CSR) and less than plan_mi's resident bytes;
    the host holds the coarsest level."""
    import ctypes as C
    from paper_2007_00056_b200 import _lib
    A = sp.graph_laplacian3d(24, seed=5)  # general values: SELL-G / CSR levels, not row patterns
    cfg = _cfg(sp)
    L = sp.Hierarchy(A, cfg).nlevels()
    hh = sp.Hierarchy(A, cfg, host_levels_from=L - 1)
    rh = ref.hierarchy(A, 500, 40)
    assert rh.nlevels() == L
    _, mi_resident, mi_cycle = rh.memory_plan("MI")
    on_host, mb = C.c_int(), C.c_int64()
    dev_mat = dev_csr = 0
    for k in range(L):
        _lib.check(_lib.lib().sb_level_residency(hh.ctx(), k, C.byref(on_host), C.byref(mb)))
        assert on_host.value == (1 if k == L - 1 else 0), k
        assert mb.value <= 1.25 * rh.csr_bytes(k), (k, mb.value, rh.csr_bytes(k))
        if not on_host.value:
            dev_mat += mb.value
            dev_csr += rh.csr_bytes(k)
    assert dev_mat <= dev_csr
    assert dev_mat < mi_resident
    _lib.check(_lib.lib().sb_level_residency(hh.ctx(), L - 1, C.byref(on_host), C.byref(mb)))
    assert hh.host_bytes() >= mb.value > 0
    # MI moves only the coarse rhs down and the coarse solution up per cycle
    nc = rh.level(L - 1)[0].size - 1
    assert mi_cycle == 2 * 8 * nc
