"""Single-kernel parity on the GPU through the C ABI: SpMV, residual, Jacobi
sweeps, restriction and prolongation are bit-identical to the reference
(thread-per-row CSR-order sums, no FMA); the coarse solve uses a precomputed
inverse and matches to 1e-12 relative."""
import glob
import os

import numpy as np
import pytest

from conftest import golden_path
from helpers import from_npz, random_sparse, random_spd, rel

pytestmark = pytest.mark.gpu


def _mats(sp):
    long_row = np.zeros((40, 40))
    np.fill_diagonal(long_row, 50.0)
    long_row[3, :] = 1.0
    long_row[3, 3] = 60.0
    return [sp.poisson2d(33, 17), sp.poisson3d(20), sp.aniso3d(16), sp.poisson3d_27(9),
            sp.convdiff3d(11, 12, 13, 1.0, 100.0, 1.0, 1.0), random_sparse(sp, 70, 3, 0.3, False),
            random_spd(sp, 50, 4), sp.CsrMatrix.from_dense(long_row)]


FORMATS = [("0", "0", "0"), ("1", "0", "0"), ("0", "1", "0"), ("1", "1", "0"), ("1", "1", "1")]


@pytest.mark.parametrize("compress,sell,rpat", FORMATS)
def test_spmv_residual_bitexact(sp, oracle_best, compress, sell, rpat, monkeypatch):
    # SB_COMPRESS=1 (default): dictionary values + int16 column deltas where
    # they fit; SB_SELL=1 (default): grouped sliced-ELL slices; SB_RPAT=1
    # (default): one pattern byte per row where a level has <= 256 distinct
    # rows. All must give the reference's bits.
    monkeypatch.setenv("SB_COMPRESS", compress)
    monkeypatch.setenv("SB_SELL", sell)
    monkeypatch.setenv("SB_RPAT", rpat)
    mats = _mats(sp) + [sp.stencil7(200, 200, 2, 6.0, [-1.0] * 6)]  # |delta| 40000: int32 columns
    for A in mats:
        x = np.random.default_rng(1).uniform(-1, 1, A.ncols())
        f = np.random.default_rng(2).uniform(-1, 1, A.nrows())
        assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x))
        assert np.array_equal(sp.residual(A, x, f), oracle_best.residual(A, x, f))


def test_spmv_long_rows_unstaged_path(sp, oracle_best):
    # a row with > 8192 entries exceeds the per-tile staging capacity
    n = 9000
    ent = [(i, i, 4.0) for i in range(n)] + [(7, j, 0.5 + (j % 3)) for j in range(n) if j != 7]
    A = sp.CsrMatrix.from_triplets(n, n, ent)
    x = np.random.default_rng(5).uniform(-1, 1, n)
    assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x))


@pytest.mark.parametrize("sweeps", [1, 2, 3, 6])
@pytest.mark.parametrize("compress,sell,rpat", FORMATS)
def test_jacobi_bitexact(sp, oracle_best, sweeps, compress, sell, rpat, monkeypatch):
    monkeypatch.setenv("SB_COMPRESS", compress)
    monkeypatch.setenv("SB_SELL", sell)
    monkeypatch.setenv("SB_RPAT", rpat)
    jac = sp.SmootherKind.weighted_jacobi()
    for A in _mats(sp):
        x = np.random.default_rng(3).uniform(-1, 1, A.nrows())
        f = np.random.default_rng(4).uniform(-1, 1, A.nrows())
        got = sp.smooth(jac, A, x, f, sweeps)
        assert np.array_equal(got, oracle_best.jacobi(A, 2.0 / 3.0, x, f, sweeps))


def test_jacobi_hand_values(sp):
    # test_smoother.cpp:33-51
    D = sp.CsrMatrix.from_dense([[2, 0, 0], [0, 4, 0], [0, 0, 8]])
    x = sp.smooth(sp.SmootherKind.weighted_jacobi(1.0), D, np.zeros(3), [2.0, 2.0, 2.0], 1)
    assert x.tolist() == [1.0, 0.5, 0.25]
    A = sp.CsrMatrix.from_dense([[2, 1], [1, 3]])
    x = sp.smooth(sp.SmootherKind.weighted_jacobi(0.5), A, [1.0, -1.0], [3.0, 2.0], 1)
    assert x[0] == 1.5 and x[1] == -1.0 + 2.0 / 3.0


def test_jacobi_fixed_point_and_errors(sp):
    # test_smoother.cpp:114-125: integer data, exact solution is a fixed point
    A = sp.poisson2d(4, 4)
    x = np.array([float(i % 5 - 2) for i in range(16)])
    f = sp.spmv(A, x)
    assert np.array_equal(sp.smooth(sp.SmootherKind.weighted_jacobi(), A, x, f, 4), x)
    # test_smoother.cpp:170-186: zero / missing diagonal reported with the row
    Z = sp.CsrMatrix.from_triplets(2, 2, [(0, 0, 1.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 0.0)])
    with pytest.raises(sp.InvalidArgument, match="row 1"):
        sp.smooth(sp.SmootherKind.weighted_jacobi(), Z, np.zeros(2), [1.0, 1.0], 1)
    with pytest.raises(sp.InvalidArgument, match="Jacobi"):
        sp.smooth(sp.SmootherKind.gauss_seidel_forward(), A, np.zeros(16), np.ones(16), 1)
    assert np.array_equal(sp.smooth(sp.SmootherKind.weighted_jacobi(), A, x, f, 0), x)


def test_restrict_prolong_bitexact(sp):
    # test_cycle.cpp:76-100: restriction == aggregate sums (ascending), prolongation scatters
    A = sp.poisson3d(16)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40))
    for k in range(h.nlevels() - 1):
        lv = h.level(k)
        r = np.random.default_rng(k).uniform(-1, 1, lv.A.nrows())
        man = np.zeros(lv.agg.n_coarse)
        for i, c in enumerate(lv.agg.fine_to_coarse):
            man[c] += 1.0 * r[i]
        assert np.array_equal(h.restrict(k, r), man)
        xc = np.random.default_rng(100 + k).uniform(-1, 1, lv.agg.n_coarse)
        x = np.random.default_rng(200 + k).uniform(-1, 1, lv.A.nrows())
        want = x + (0.0 + xc[lv.agg.fine_to_coarse])
        assert np.array_equal(h.prolong_add(k, xc, x), want)


def test_coarse_solve(sp, oracle_best):
    A = sp.poisson3d(24)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40))
    o = oracle_best.hierarchy(A, 500, 40)
    f = np.random.default_rng(9).uniform(-1, 1, h.coarsest().nrows())
    assert rel(h.coarse_solve(f), o.coarse_solve(f)) < 1e-12


@pytest.mark.parametrize("path", sorted(p for p in glob.glob(golden_path("*.npz"))
                                        if not p.endswith("example_6x6.npz") and "config_" not in p))
def test_golden_kernels(sp, path):
    d = np.load(path)
    A = from_npz(sp, d)
    assert np.array_equal(sp.spmv(A, d["f"]), d["spmv_f"])
    assert np.array_equal(sp.smooth(sp.SmootherKind.weighted_jacobi(), A, d["f"], d["b"], 3), d["jacobi3"])


@pytest.mark.parametrize("rpat", ["0", "1"])
def test_spmv_nonfinite_inputs(sp, oracle_best, rpat, monkeypatch):
    # padded slots (boundary rows) must not turn an inf of the row's own x into
    # NaN: the pattern kernel replays such rows with masked slots
    monkeypatch.setenv("SB_RPAT", rpat)
    for A in [sp.poisson2d(24, 20), sp.poisson3d(12), sp.poisson3d_27(7)]:
        x = np.random.default_rng(8).uniform(-1, 1, A.ncols())
        x[[0, 5, A.ncols() - 1]] = [np.inf, -np.inf, np.inf]
        x[17] = np.nan
        f = np.random.default_rng(9).uniform(-1, 1, A.nrows())
        got, want = sp.spmv(A, x), oracle_best.spmv(A, x)
        assert np.array_equal(got, want, equal_nan=True)
        assert np.array_equal(np.signbit(got), np.signbit(want))
        assert np.array_equal(sp.residual(A, x, f), oracle_best.residual(A, x, f), equal_nan=True)


@pytest.mark.parametrize("dims", [(100, 4, 3), (128, 5, 4), (96, 3, 2)])
def test_27point_varied_bitexact(sp, oracle_best, dims):
    # 27-point rows (the wide row-pattern path, W = 28) with a different value
    # per direction: any slip in slot order or value/column pairing changes bits
    from helpers import stencil27_varied
    A = stencil27_varied(sp, *dims, seed=sum(dims))
    x = np.random.default_rng(11).uniform(-1, 1, A.ncols())
    f = np.random.default_rng(12).uniform(-1, 1, A.nrows())
    assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x))
    assert np.array_equal(sp.residual(A, x, f), oracle_best.residual(A, x, f))
    jac = sp.SmootherKind.weighted_jacobi()
    assert np.array_equal(sp.smooth(jac, A, x, f, 3), oracle_best.jacobi(A, 2.0 / 3.0, x, f, 3))
    x[[40, 41, 200]] = [np.inf, np.nan, -np.inf]  # non-finite values inside interior rows
    assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x), equal_nan=True)


@pytest.mark.parametrize("case", ["many-in-one-tile", "spread", "longer-than-buffer"])
def test_csr_tile_long_rows_cta_path(sp, oracle_best, case, monkeypatch):
    """k_csr_tile defers rows of > 32 entries (up to 16 per CTA) to the end of
    the kernel, where the whole CTA forms their products and one thread per row
    adds them in CSR order; more rows per CTA take the warp path, and a row
    longer than the drained stage buffers is added segment by segment. SpMV,
    residual and Jacobi must stay the reference's bits in every case."""
    monkeypatch.setenv("SB_SELL", "0")
    monkeypatch.setenv("SB_RPAT", "0")
    rng = np.random.default_rng({"many-in-one-tile": 1, "spread": 2, "longer-than-buffer": 3}[case])
    n = {"many-in-one-tile": 600, "spread": 3000, "longer-than-buffer": 9000}[case]
    hubs = {"many-in-one-tile": list(range(10, 240, 10)),            # 23 long rows in the first tile
            "spread": list(rng.choice(n, 40, replace=False)),         # long rows across many tiles
            "longer-than-buffer": [5, 4000]}[case]                    # rows with ~n entries
    ent = {}
    for i in range(n):
        ent[(i, i)] = 4.0
        for j in (i - 1, i + 1):
            if 0 <= j < n:
                ent[(i, j)] = -1.0
    for h in hubs:
        cols = np.arange(n) if case == "longer-than-buffer" else rng.choice(n, int(rng.integers(33, 400)),
                                                                              replace=False)
        for j in cols:
            if j != h:
                ent[(int(h), int(j))] = -float(rng.uniform(0.001, 0.01))
        ent[(int(h), int(h))] = 4.0 + float(len(cols)) * 0.01
    A = sp.CsrMatrix.from_triplets(n, n, [(r, c, v) for (r, c), v in ent.items()])
    x = rng.uniform(-1, 1, n)
    f = rng.uniform(-1, 1, n)
    assert np.array_equal(sp.spmv(A, x), oracle_best.spmv(A, x))
    assert np.array_equal(sp.residual(A, x, f), oracle_best.residual(A, x, f))
    jac = sp.SmootherKind.weighted_jacobi()
    assert np.array_equal(sp.smooth(jac, A, x, f, 3), oracle_best.jacobi(A, 2.0 / 3.0, x, f, 3))
