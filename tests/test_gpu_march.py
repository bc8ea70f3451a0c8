"""Plane-marching row-pattern sweep (k_march, csrc/sb_march.cuh): on levels whose
main pattern is a 27-point box, a CTA stages the x planes of
an 8-line x 32-column tile in shared memory by TMA and rolls each row's gathered
values in registers from plane to plane. Every result must stay bit-identical
to the reference (inc/csr.hpp:174-194, 267-274, inc/smoother.hpp:113-120):
boundary rows embedded into the main slot order, absent slots that read
inf/NaN (exact replay), ragged tiles, first / last planes (per-row path), and
whole V-cycles, which must equal the non-marching path bit for bit."""
import ctypes as C

import numpy as np
import pytest

from conftest import needs_experimental

from helpers import stencil27_varied

pytestmark = pytest.mark.gpu


def _march(sp, A_or_h, level=0):
    from paper_2007_00056_b200 import _lib
    h = A_or_h._device() if isinstance(A_or_h, sp.CsrMatrix) else A_or_h
    g, s = C.c_int(), C.c_int()
    _lib.check(_lib.lib().sb_level_march(h.ctx(), level, C.byref(g), C.byref(s)))
    return g.value, s.value


def _p27(sp, nx, ny, nz):
    from paper_2007_00056_b200 import _lib
    return sp._gen(_lib.lib().sb_gen_stencil27, nx, ny, nz, 26.0, -1.0)


def _cases(sp):
    # march tiles are 32 columns x 8 lines x 16 planes: ragged column / line
    # blocks, fewer and more planes than a tile, several tiles per CTA
    return [
        ("box27", lambda: _p27(sp, 40, 9, 40), 0),
        ("box27-varied", lambda: stencil27_varied(sp, 37, 11, 9, seed=3), 0),
        ("box27-varied-wide", lambda: stencil27_varied(sp, 64, 6, 5, seed=4), 0),
        ("box27-varied-deep", lambda: stencil27_varied(sp, 33, 17, 36, seed=5), 0),
        # 7-point levels keep the row-pattern kernel (measured faster there)
        ("cross7", lambda: sp.poisson3d(33, 10, 40), -1),
        ("cross7-aniso", lambda: sp.stencil7(45, 13, 21, 4.002, [-1.0, -1.0, -1.0, -1.0, -1e-3, -1e-3]), -1),
        ("cross7-convdiff", lambda: sp.convdiff3d(36, 9, 20, 1.0, 100.0, 1.0, 1.0), -1),
        ("cross5-none", lambda: sp.poisson2d(45, 29), -1),
    ]


@needs_experimental
@pytest.mark.parametrize("idx", range(8))
def test_march_kernels_bitexact(sp, oracle_best, idx, monkeypatch):
    monkeypatch.setenv("SB_BOXPAIR", "0")
    monkeypatch.setenv("SB_MARCH", "1")
    monkeypatch.setenv("SB_MARCH_MIN", "0")
    name, make, geo = _cases(sp)[idx]
    A = make()
    assert _march(sp, A)[0] == geo, name
    n = A.nrows()
    rng = np.random.default_rng(idx)
    x = rng.uniform(-1, 1, n)
    f = rng.uniform(-1, 1, n)
    assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x)), name
    assert np.array_equal(sp.residual(A, x, f), oracle_best.residual(A, x, f)), name
    jac = sp.SmootherKind.weighted_jacobi()
    for sweeps in (1, 4):
        assert np.array_equal(sp.smooth(jac, A, x, f, sweeps), oracle_best.jacobi(A, 2.0 / 3.0, x, f, sweeps)), name


@pytest.mark.parametrize("kern", ["march", "boxpair"])
@pytest.mark.parametrize("idx", [0, 1, 2, 3])
def test_march_nonfinite_absent_slots(sp, oracle_best, idx, kern, monkeypatch):
    # inf / NaN at x positions that boundary rows read only through absent
    # (embedded +0.0 / masked) slots: 0 * inf would be NaN
    monkeypatch.setenv("SB_BOXPAIR", "1" if kern == "boxpair" else "0")
    monkeypatch.setenv("SB_MARCH", "1" if kern == "march" else "0")
    monkeypatch.setenv("SB_MARCH_MIN", "0")
    _, make, _ = _cases(sp)[idx]
    A = make()
    n = A.nrows()
    x = np.random.default_rng(7).uniform(-1, 1, n)
    rp = A.row_ptr()
    lens = np.diff(rp)
    short = np.nonzero(lens < lens.max())[0]  # boundary rows
    pick = short[len(short) // 3:len(short) // 3 + 40]
    for j, r in enumerate(pick[::4]):
        for c in (r - 1, r + 1):  # neighbours that are not in the row but inside [0, n)
            if 0 <= c < n:
                x[c] = [np.inf, -np.inf, np.nan][j % 3]
    f = np.random.default_rng(8).uniform(-1, 1, n)
    got, want = sp.spmv(A, x), oracle_best.spmv(A, x)
    assert np.array_equal(got, want, equal_nan=True)
    # NaN made by an invalid operation (inf - inf) has the platform's default
    # sign (the GPU's differs from x86's); compare signs of the numbers
    num = ~np.isnan(want)
    assert np.array_equal(np.signbit(got[num]), np.signbit(want[num]))
    jac = sp.SmootherKind.weighted_jacobi()
    assert np.array_equal(sp.smooth(jac, A, x, f, 1), oracle_best.jacobi(A, 2.0 / 3.0, x, f, 1), equal_nan=True)


def _solve(sp, A, march, monkeypatch):
    monkeypatch.setenv("SB_BOXPAIR", "0")
    monkeypatch.setenv("SB_MARCH", "1" if march else "0")
    monkeypatch.setenv("SB_MARCH_MIN", "0")
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
    h = sp.Hierarchy(A, cfg, device=0)
    geos = [_march(sp, h, k)[0] for k in range(h.nlevels())]
    b = sp.rhs_ones(A.nrows())
    cp = sp.CycleParams.from_config(cfg)
    v = sp.vcycle(h, 0, b, np.zeros(A.nrows()), cp)
    res = sp.pcg(A, b, sp.make_amg_preconditioner(h, cp), 1e-8 * float(np.linalg.norm(b)), 200)
    return geos, v, res


@needs_experimental
@pytest.mark.parametrize("dims", [(48, 16, 40), (45, 13, 37)])  # even / odd line and plane strides
def test_march_vcycle_pcg_identical(sp, dims, monkeypatch):
    A = _p27(sp, *dims)
    g1, v1, r1 = _solve(sp, A, True, monkeypatch)
    g0, v0, r0 = _solve(sp, A, False, monkeypatch)
    assert max(g1) >= 0 and max(g0) == -1
    assert np.array_equal(v1, v0)
    # the V-cycle is bitwise the same; the fused dot products reduce in another
    # per-thread order (deterministic, rounding-level differences)
    assert r1.report.iterations == r0.report.iterations
    assert np.linalg.norm(r1.x - r0.x) <= 1e-12 * np.linalg.norm(r0.x)


# ---- k_boxpair (sb_rowpat.cuh): row pairs with 16-byte loads on 27-point box
# levels whose line / plane strides are even (the default kernel there) -------

def _sweep_kernel(sp, A_or_h, level=0):
    from paper_2007_00056_b200 import _lib
    h = A_or_h._device() if isinstance(A_or_h, sp.CsrMatrix) else A_or_h
    buf = C.create_string_buffer(64)
    _lib.check(_lib.lib().sb_level_sweep_kernel(h.ctx(), level, buf, 64))
    return buf.value.decode()


@pytest.mark.parametrize("case", ["p27", "varied", "varied-odd", "poisson7", "convdiff7", "aniso7-odd",
                                  "poisson5", "poisson5-odd"])
def test_boxpair_kernels_bitexact(sp, oracle_best, case, monkeypatch):
    # k_boxpair (27-point box) / k_crosspair (7- and 5-point cross): row pairs,
    # 16-byte loads, restriction masks for boundary rows; odd strides keep k_rowpat
    monkeypatch.setenv("SB_BOXPAIR", "1")
    monkeypatch.setenv("SB_CROSS5", "1")
    A, want_k = {"p27": (lambda: _p27(sp, 40, 10, 40), "k_boxpair"),
                 "varied": (lambda: stencil27_varied(sp, 64, 6, 9, seed=8), "k_boxpair"),
                 "varied-odd": (lambda: stencil27_varied(sp, 33, 17, 12, seed=9), "k_rowpat"),  # odd N
                 "poisson7": (lambda: sp.poisson3d(34, 12, 20), "k_crosspair"),
                 "convdiff7": (lambda: sp.convdiff3d(36, 10, 14, 1.0, 100.0, 1.0, 1.0), "k_crosspair"),
                 "aniso7-odd": (lambda: sp.stencil7(45, 13, 21, 4.002, [-1.0, -1.0, -1.0, -1.0, -1e-3, -1e-3]),
                                "k_rowpat"),
                 "poisson5": (lambda: sp.poisson2d(46, 30), "k_crosspair"),
                 "poisson5-odd": (lambda: sp.poisson2d(45, 29), "k_rowpat")}[case]
    A = A()
    assert _sweep_kernel(sp, A) == want_k
    n = A.nrows()
    rng = np.random.default_rng(21)
    x = rng.uniform(-1, 1, n)
    f = rng.uniform(-1, 1, n)
    assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x))
    assert np.array_equal(sp.residual(A, x, f), oracle_best.residual(A, x, f))
    jac = sp.SmootherKind.weighted_jacobi()
    for sweeps in (1, 4):
        assert np.array_equal(sp.smooth(jac, A, x, f, sweeps), oracle_best.jacobi(A, 2.0 / 3.0, x, f, sweeps))
    x[[n // 2, n // 3, 5]] = [np.inf, np.nan, -np.inf]  # interior (pair path) and boundary rows
    assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x), equal_nan=True)


@pytest.mark.parametrize("which", ["p27", "p7", "p5"])
def test_boxpair_vcycle_pcg_identical(sp, which, monkeypatch):
    A = {"p27": lambda: _p27(sp, 48, 16, 40), "p7": lambda: sp.poisson3d(64, 40, 40),
         "p5": lambda: sp.poisson2d(256, 200)}[which]()
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
    b = sp.rhs_ones(A.nrows())
    cp = sp.CycleParams.from_config(cfg)
    monkeypatch.setenv("SB_CROSS5", "1")
    out = {}
    for on in ("1", "0"):
        monkeypatch.setenv("SB_BOXPAIR", on)
        h = sp.Hierarchy(A, cfg, device=0)
        ks = [_sweep_kernel(sp, h, k) for k in range(h.nlevels() - 1)]
        v = sp.vcycle(h, 0, b, np.zeros(A.nrows()), cp)
        r = sp.pcg(A, b, sp.make_amg_preconditioner(h, cp), 1e-8 * float(np.linalg.norm(b)), 200)
        out[on] = (ks, v, r)
    pair = "k_boxpair" if which == "p27" else "k_crosspair"
    assert pair in out["1"][0] and pair not in out["0"][0]
    assert np.array_equal(out["1"][1], out["0"][1])
    assert out["1"][2].report.iterations == out["0"][2].report.iterations
    assert np.linalg.norm(out["1"][2].x - out["0"][2].x) <= 1e-12 * np.linalg.norm(out["0"][2].x)


@needs_experimental
def test_cross_rr_vcycle_identical():
    # k_cross_rr (opt-in, read once per process): residual + restriction from row
    # pairs gives bitwise the same V-cycle as k_pat_resid_restrict
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np; sys.path.insert(0, %r); from paper_2007_00056_b200 import sparsh as sp; "
            "A = sp.poisson3d(64, 40, 40); "
            "cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40); "
            "h = sp.Hierarchy(A, cfg); b = sp.rhs_random(A.nrows(), 5); "
            "v = sp.vcycle(h, 0, b, np.zeros(A.nrows()), sp.CycleParams.from_config(cfg)); "
            "sys.stdout.write(v.tobytes().hex())") % root
    vs = []
    for on in ("1", "0"):
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SB_CROSS_RR=on), capture_output=True,
                             text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        vs.append(out.stdout)
    assert vs[0] and vs[0] == vs[1]


def test_cross5_default_selection(sp, monkeypatch):
    """Default 5-point selection (SB_CROSS5 unset): the pair kernel on 2D levels
    of >= 2^19 rows only (k_crosspair at L0 of a 1024x512 grid, k_rowpat at L1);
    the V-cycle is bitwise the one with the pair kernel off everywhere."""
    A = sp.poisson2d(1024, 512)
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
    cp = sp.CycleParams.from_config(cfg)
    f = sp.rhs_random(A.nrows(), 4)
    monkeypatch.delenv("SB_CROSS5", raising=False)
    h = sp.Hierarchy(A, cfg)
    assert _sweep_kernel(sp, h, 0) == "k_crosspair" and _sweep_kernel(sp, h, 1) == "k_rowpat"
    v = sp.vcycle(h, 0, f, np.zeros(A.nrows()), cp)
    monkeypatch.setenv("SB_CROSS5", "0")
    h0 = sp.Hierarchy(A, cfg)
    assert _sweep_kernel(sp, h0, 0) == "k_rowpat"
    v0 = sp.vcycle(h0, 0, f, np.zeros(A.nrows()), cp)
    assert np.array_equal(v.view(np.uint64), v0.view(np.uint64))
