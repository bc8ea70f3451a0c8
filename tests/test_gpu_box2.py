"""Two Jacobi sweeps per launch (k_cross_box2, csrc/sb_box2.cuh; built with
make EXPERIMENTAL=1, enabled with SB_BOX2=1) on mid-size structured 7-point levels: bitwise equal to the reference's sweeps
(inc/smoother.hpp:95-123) for any sweep count, including non-finite inputs
and levels whose tiles / z-chunks do not divide the grid; V-cycles and whole
solves bitwise equal to the unfused path (SB_BOX2=0)."""
import ctypes as C

import numpy as np
import pytest

from helpers import rel

from conftest import needs_experimental

pytestmark = [pytest.mark.gpu, needs_experimental]


@pytest.fixture(autouse=True)
def _box_all(monkeypatch):
    monkeypatch.setenv("SB_BOX2", "1")  # opt-in (measured slower)
    monkeypatch.setenv("SB_BOX2_MIN", "0")  # every structured level of these small grids takes it

GRIDS = {
    "poisson3d_24": lambda sp: sp.poisson3d(24),
    "poisson3d_70x18x9": lambda sp: sp.stencil7(70, 18, 9, 6.0, [-1.0] * 6),        # partial tiles in x, ny < 16
    "aniso3d_20": lambda sp: sp.aniso3d(20, 1e-3),
    "convdiff3d_16x18x22": lambda sp: sp.convdiff3d(16, 18, 22, 1.0, 100.0, 1.0, 1.0),  # distinct +/- values
    "poisson3d_130x34x40": lambda sp: sp.stencil7(130, 34, 40, 6.0, [-1.0] * 6),   # partial boxes in x, y, z
    "poisson3d_10x12x9": lambda sp: sp.stencil7(10, 12, 9, 6.0, [-1.0] * 6),      # 8-wide boxes, ny < 16
}


def _fused(sp, h, k):
    from paper_2007_00056_b200 import _lib
    geo = (C.c_int * 8)()
    return _lib.lib().sb_level_fused_sweeps(h.ctx(), k, geo), list(geo)


def _cfg(sp):
    return sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)


@pytest.mark.parametrize("name", sorted(GRIDS))
@pytest.mark.parametrize("sweeps", [1, 2, 3, 4, 5])
def test_fused_sweeps_bitexact(sp, oracle_best, name, sweeps):
    A = GRIDS[name](sp)
    n = A.nrows()
    h = sp.Hierarchy(A, _cfg(sp))
    assert _fused(sp, h, 0)[0] == 2, "level 0 must take the fused kernel"
    rng = np.random.default_rng(sweeps)
    x = rng.uniform(-1, 1, n)
    f = rng.uniform(-1, 1, n)
    out = h.smooth(0, sp.SmootherKind.weighted_jacobi(), x, f, sweeps)
    ref = oracle_best.jacobi(A, 2.0 / 3.0, x, f, sweeps)
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("name", ["poisson3d_24", "convdiff3d_16x18x22"])
def test_fused_sweeps_nonfinite(sp, oracle_best, name):
    A = GRIDS[name](sp)
    n = A.nrows()
    h = sp.Hierarchy(A, _cfg(sp))
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, n)
    f = rng.uniform(-1, 1, n)
    # boundary rows (corners, faces) and interior rows
    x[[0, 1, n - 1, n // 2, n // 2 + 7, 40]] = [np.inf, -np.inf, np.nan, np.inf, np.nan, -np.inf]
    f[[5, n - 3]] = [np.nan, np.inf]
    for sweeps in (2, 4):
        out = h.smooth(0, sp.SmootherKind.weighted_jacobi(), x, f, sweeps)
        ref = oracle_best.jacobi(A, 2.0 / 3.0, x, f, sweeps)
        # NaN payloads differ between x86 and the GPU; every other bit must match
        assert np.array_equal(np.isnan(out), np.isnan(ref))
        ok = ~np.isnan(ref)
        assert np.array_equal(out[ok].view(np.uint64), ref[ok].view(np.uint64))
        assert np.isinf(ref).any() and np.isnan(ref).any()


@pytest.mark.parametrize("name", sorted(GRIDS))
def test_fused_vcycle_and_pcg_equal_unfused(sp, monkeypatch, name):
    A = GRIDS[name](sp)
    b = sp.rhs_random(A.nrows(), 42)
    tol = 1e-8 * np.linalg.norm(b)
    cp = sp.CycleParams.from_config(_cfg(sp))
    out = {}
    for tb in ("1", "0"):
        monkeypatch.setenv("SB_BOX2", tb)
        h = sp.Hierarchy(A, _cfg(sp))
        nf = [_fused(sp, h, k)[0] for k in range(h.nlevels())]
        v = sp.vcycle(h, 0, b, np.zeros(A.nrows()), cp)
        solver = sp.pbicgstab if "convdiff" in name else sp.pcg
        r = solver(A, b, sp.make_amg_preconditioner(h, cp), tol, 200)
        out[tb] = (nf, v, r)
    assert out["1"][0][0] == 2 and all(k == 1 for k in out["0"][0])
    assert np.array_equal(out["1"][1].view(np.uint64), out["0"][1].view(np.uint64))
    r1, r0 = out["1"][2], out["0"][2]
    assert r1.report.iterations == r0.report.iterations
    assert np.array_equal(r1.x.view(np.uint64), r0.x.view(np.uint64))


def test_fused_vcycle_vs_reference(sp, oracle_best):
    """One V-cycle with the fused sweeps on every structured level vs the reference
    (coarse_exact: the reference's substitution order -> bitwise)."""
    A = sp.poisson3d(32)
    h = sp.Hierarchy(A, _cfg(sp), coarse_exact=True)
    assert sum(_fused(sp, h, k)[0] == 2 for k in range(h.nlevels())) >= 3
    f = sp.rhs_random(A.nrows(), 7)
    v = sp.vcycle(h, 0, f, np.zeros(A.nrows()), sp.CycleParams.from_config(_cfg(sp)))
    o = oracle_best.hierarchy(A, 500, 40)
    ref = o.vcycle(f, np.zeros(A.nrows()))
    assert np.array_equal(v.view(np.uint64), ref.view(np.uint64))
