"""V-cycle parity on the GPU (cycle.hpp:53-75): every level operation is
bitwise the reference's except the coarsest solve (inverse GEMV), so one
V-cycle agrees to ~1e-15; the contract is 1e-12 relative."""
import numpy as np
import pytest

from helpers import random_spd, rel

pytestmark = pytest.mark.gpu

JAC = None


def _cp(sp, pre=6, post=6, omega=2.0 / 3.0):
    return sp.CycleParams(pre, post, sp.SmootherKind.weighted_jacobi(omega))


@pytest.mark.parametrize("mk", [
    lambda sp: sp.poisson3d(32), lambda sp: sp.aniso3d(24), lambda sp: sp.poisson2d(96, 80),
    lambda sp: sp.convdiff3d(16, 16, 16, 1.0, 100.0, 1.0, 1.0), lambda sp: sp.poisson3d_27(12),
    lambda sp: random_spd(sp, 300, 7, 0.05)])
@pytest.mark.parametrize("sweeps", [(6, 6), (1, 2), (0, 3), (2, 0), (3, 5)])
@pytest.mark.parametrize("tail_rows,compress,sell,rpat", [
    ("0", "0", "0", "0"), ("0", "1", "0", "0"), ("0", "0", "1", "0"), ("0", "1", "1", "0"), ("0", "1", "1", "1"),
    ("2000", "1", "1", "1"), ("1048576", "1", "1", "1"), ("1048576", "1", "1", "0")])
def test_vcycle_matches_oracle(sp, port, mk, sweeps, tail_rows, compress, sell, rpat, monkeypatch):
    # SB_TAIL_ROWS=0: every level as separate kernels; otherwise the small
    # levels run inside the cluster-resident tail kernel. SB_COMPRESS / SB_SELL /
    # SB_RPAT toggle the lossless streamed matrix formats.
    monkeypatch.setenv("SB_TAIL_ROWS", tail_rows)
    monkeypatch.setenv("SB_COMPRESS", compress)
    monkeypatch.setenv("SB_SELL", sell)
    monkeypatch.setenv("SB_RPAT", rpat)
    A = mk(sp)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40, coarse_target=min(500, A.nrows() // 4)))
    o = port.hierarchy(A, min(500, A.nrows() // 4), 40)
    o.set_cycle(sweeps[0], sweeps[1], 2.0 / 3.0)
    cp = _cp(sp, *sweeps)
    f = sp.rhs_random(A.nrows(), 42)
    got = sp.vcycle(h, 0, f, np.zeros(A.nrows()), cp)
    assert rel(got, o.vcycle(f, np.zeros(A.nrows()))) < 1e-12
    # the preconditioner path (x = 0 promise, fused first sweeps, tail)
    assert rel(sp.make_amg_preconditioner(h, cp).apply(f), o.vcycle(f, np.zeros(A.nrows()))) < 1e-12
    x0 = np.random.default_rng(1).uniform(-1, 1, A.nrows())  # general initial guess
    assert rel(sp.vcycle(h, 0, f, x0, cp), o.vcycle(f, x0)) < 1e-12


def test_vcycle_linear_symmetric_zero(sp):
    # test_cycle.cpp:32-56, 188-199
    h = sp.Hierarchy(sp.poisson2d(16, 16), sp.SolverConfig(coarse_target=60))
    cp = _cp(sp)
    rng = np.random.default_rng(83)
    f, g = rng.uniform(-1, 1, 256), rng.uniform(-1, 1, 256)
    Bf, Bg = sp.vcycle(h, 0, f, np.zeros(256), cp), sp.vcycle(h, 0, g, np.zeros(256), cp)
    Bc = sp.vcycle(h, 0, 2 * f - 3 * g, np.zeros(256), cp)
    assert np.max(np.abs(Bc - (2 * Bf - 3 * Bg))) <= 1e-10 * np.max(np.abs(Bc))
    M = sp.make_amg_preconditioner(h, cp)
    for _ in range(10):
        u, v = rng.uniform(-1, 1, 256), rng.uniform(-1, 1, 256)
        a, b = M.apply(u) @ v, u @ M.apply(v)
        assert abs(a - b) <= 1e-9 * max(1.0, abs(a))
    assert not sp.vcycle(h, 0, np.zeros(256), np.zeros(256), cp).any()
    assert np.array_equal(M.apply(f), sp.vcycle(h, 0, f, np.zeros(256), cp))


def test_residual_drops_every_cycle(sp):
    # test_cycle.cpp:58-72 (Jacobi variant)
    A = sp.poisson2d(64, 64)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40))
    b = sp.rhs_ones(4096)
    x = np.zeros(4096)
    prev = np.linalg.norm(b)
    for _ in range(5):
        sp.vcycle_in_place(h, 0, b, x, _cp(sp))
        rn = np.linalg.norm(sp.residual(A, x, b))
        assert rn < prev
        prev = rn


def test_single_level_is_direct_solve(sp):
    A = sp.CsrMatrix.from_dense([[4, -1, 0], [-1, 4, -1], [0, -1, 4]])
    h = sp.Hierarchy(A, sp.SolverConfig(coarse_target=100))
    assert h.nlevels() == 1
    f = np.ones(3)
    assert rel(sp.vcycle(h, 0, f, np.zeros(3), _cp(sp)), np.linalg.solve(A.to_dense(), f)) < 1e-14


def test_vcycle_rejects(sp):
    h = sp.Hierarchy(sp.poisson2d(16, 16), sp.SolverConfig(coarse_target=60))
    with pytest.raises(sp.InvalidArgument):
        sp.vcycle(h, 0, np.ones(255), np.zeros(256), _cp(sp))
    with pytest.raises(sp.InvalidArgument, match="Jacobi"):
        sp.vcycle(h, 0, np.ones(256), np.zeros(256), sp.CycleParams())  # GS default: rejected


@pytest.mark.parametrize("tail_rows", ["0", "32768"])
def test_vcycle_bitexact_with_exact_coarse(sp, port, tail_rows, monkeypatch):
    # with the reference-order coarse substitution every level is bitwise the
    # reference's (the tail is disabled in that mode)
    monkeypatch.setenv("SB_TAIL_ROWS", tail_rows)
    A = sp.poisson3d(24)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40), coarse_exact=True)
    o = port.hierarchy(A, 500, 40)
    f = sp.rhs_random(A.nrows(), 3)
    assert np.array_equal(sp.vcycle(h, 0, f, np.zeros(A.nrows()), _cp(sp)), o.vcycle(f, np.zeros(A.nrows())))


@pytest.mark.parametrize("tail_rows", ["0", "8192"])
def test_vcycle_27point_varied_bitexact(sp, port, tail_rows, monkeypatch):
    # direction-weighted 27-point operator (wide row patterns on every level);
    # with the reference-order coarse solve the whole cycle is bitwise the
    # reference's
    from helpers import stencil27_varied
    monkeypatch.setenv("SB_TAIL_ROWS", tail_rows)
    for dims in [(96, 6, 5), (128, 4, 4)]:
        A = stencil27_varied(sp, *dims, seed=3)
        h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40, coarse_target=64), coarse_exact=True)
        o = port.hierarchy(A, 64, 40)
        f = sp.rhs_random(A.nrows(), 5)
        assert np.array_equal(sp.vcycle(h, 0, f, np.zeros(A.nrows()), _cp(sp)), o.vcycle(f, np.zeros(A.nrows())))
        assert np.array_equal(sp.make_amg_preconditioner(h, _cp(sp)).apply(f), o.vcycle(f, np.zeros(A.nrows())))


@pytest.mark.parametrize("which", ["p3", "p2", "cd", "p3odd"])
def test_pair_paths_bitwise(sp, which):
    """Row-pair levels: residual + restriction through k_crosspair when the
    aggregates are the row pairs (SB_PAIR_RR), the prolongation folded into
    k_crosspair's first post-sweep (SB_PAIR_PC), the split prolongation
    (k_prolong2 + sweeps, SB_PROLONG_SPLIT) and k_rowpat's fused prolongation:
    every combination gives the V-cycle and the PCG solve bit for bit."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import sys, numpy as np; sys.path.insert(0, %r); from paper_2007_00056_b200 import sparsh as sp; "
            "A = %s; cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40); "
            "h = sp.Hierarchy(A, cfg); cp = sp.CycleParams.from_config(cfg); b = sp.rhs_random(A.nrows(), 5); "
            "v = sp.vcycle(h, 0, b, np.zeros(A.nrows()), cp); "
            "r = sp.pcg(A, b, sp.make_amg_preconditioner(h, cp), 1e-8 * np.linalg.norm(b), 200); "
            "sys.stdout.write(v.tobytes().hex() + ' ' + r.x.tobytes().hex() + ' ' + str(h.last_solve_launches()))")
    src = {"p3": "sp.poisson3d(32)", "p2": "sp.poisson2d(128, 96)",
           "cd": "sp.convdiff3d(40, 36, 32, 1.0, 100.0, 1.0, 1.0)", "p3odd": "sp.poisson3d(34, 22, 19)"}[which]
    outs = []
    for rr, pc, split in (("1", "1", "1"), ("0", "0", "1"), ("1", "0", "0"), ("0", "1", "1")):
        env = dict(os.environ, SB_PAIR_RR=rr, SB_PAIR_PC=pc, SB_PROLONG_SPLIT=split, SB_CROSS5="1")
        out = subprocess.run([sys.executable, "-c", code % (ROOT, src)], env=env, capture_output=True, text=True,
                             timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(out.stdout.split())
    assert outs[0] and all(o[:2] == outs[0][:2] for o in outs)
    # the folded prolongation saves one launch per row-pair level and V-cycle
    assert int(outs[0][2]) < int(outs[1][2])
