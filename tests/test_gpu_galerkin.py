"""GPU Galerkin coarse operator (north star (c)): A_c = P^T A P
computed on the device must be bit-identical to the reference's
galerkin_product (inc/aggregation.hpp:92-152) -- row pointers, column order
and every value, touched-but-zero entries included."""
import numpy as np
import pytest

from conftest import golden_path
from helpers import example_6x6, from_npz, random_sparse, random_spd

pytestmark = pytest.mark.gpu


def _same_csr(a, b):
    assert np.array_equal(a.row_ptr().astype(np.int64), b.row_ptr().astype(np.int64))
    assert np.array_equal(a.col_idx(), b.col_idx())
    assert np.array_equal(a.values().view(np.uint64), b.values().view(np.uint64))  # bitwise


def _check_levels(sp, A, cfg):
    h = sp.Hierarchy(A, cfg)
    for k in range(h.nlevels() - 1):
        L = h.level(k)
        _same_csr(sp.galerkin_product_gpu(L.A, L.agg), h.level(k + 1).A)
    return h


def test_worked_example(sp):
    # acceptance.cpp:97-126: A_c = [[4,2,0],[2,12,1],[0,1,12]], nnz 7
    A = example_6x6(sp)
    agg = sp.Aggregation(np.array([0, 0, 1, 2, 1, 2], dtype=np.int32), 3)
    Ac = sp.galerkin_product_gpu(A, agg)
    assert Ac.nnz() == 7
    assert np.array_equal(Ac.to_dense(), [[4, 2, 0], [2, 12, 1], [0, 1, 12]])


@pytest.mark.parametrize("name", ["poisson2d_16.npz", "poisson3d_12.npz", "aniso3d_12.npz", "convdiff2d_24.npz",
                                  "convdiff3d_10.npz", "poisson27_8.npz"])
def test_golden_hierarchies(sp, name):
    d = np.load(golden_path(name))
    _check_levels(sp, from_npz(sp, d), sp.SolverConfig(max_levels=40))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_values(sp, seed):
    # random values make every accumulation-order difference visible in the bits
    _check_levels(sp, random_sparse(sp, 90, seed, density=0.08), sp.SolverConfig(coarse_target=4, max_levels=40))
    _check_levels(sp, random_spd(sp, 70, seed, density=0.1), sp.SolverConfig(coarse_target=4, max_levels=40))


def test_touched_zero_kept(sp):
    # (A_c)_kl sums to exactly 0.0 but is touched: stored (aggregation.hpp:143-147)
    A = sp.CsrMatrix.from_dense([[2.0, 1.0, 0.0, 0.0], [1.0, 2.0, -1.0, 0.0], [0.0, -1.0, 2.0, 1.0],
                                 [0.0, 1.0, 1.0, 2.0]])
    agg = sp.Aggregation(np.array([0, 0, 1, 1], dtype=np.int32), 2)
    Ac = sp.galerkin_product_gpu(A, agg)
    host = sp.Hierarchy(A, sp.SolverConfig(coarse_target=1, max_levels=2))
    assert Ac.nnz() == 4 and 0.0 in Ac.values().tolist()
    if host.level(0).agg.fine_to_coarse.tolist() == [0, 0, 1, 1]:
        _same_csr(Ac, host.level(1).A)


def test_setup_with_gpu_galerkin_matches_host(sp):
    A = sp.poisson3d(24)
    cfg = sp.SolverConfig(max_levels=40)
    hh = sp.Hierarchy(A, cfg)
    hg = sp.Hierarchy(A, cfg, galerkin_gpu=True)
    assert hh.nlevels() == hg.nlevels()
    for k in range(hh.nlevels()):
        _same_csr(hh.level(k).A, hg.level(k).A)
        if k + 1 < hh.nlevels():
            assert np.array_equal(hh.level(k).agg.fine_to_coarse, hg.level(k).agg.fine_to_coarse)


def test_rejects_bad_aggregation(sp):
    A = sp.poisson2d(4, 4)
    with pytest.raises(sp.InvalidArgument):
        sp.galerkin_product_gpu(A, sp.Aggregation(np.zeros(16, dtype=np.int32), 1))  # 16 fine nodes in one aggregate
