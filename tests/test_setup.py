"""Host setup of the product (node-HEM, Galerkin, coarse LU, generators) is
bit-exact with the reference (SURVEY.md §8 parity: aggregates and coarse
sparsity ==). CPU only: no device context is created."""
import numpy as np
import pytest

from helpers import example_6x6, random_sparse, random_spd


def _same_hierarchy(h, o):
    assert h.nlevels() == o.nlevels()
    for k in range(h.nlevels()):
        L = h.level(k)
        rp, ci, v, agg = o.level(k)
        assert np.array_equal(L.A.row_ptr().astype(np.int64), rp.astype(np.int64)), k
        assert np.array_equal(L.A.col_idx(), ci), k
        assert np.array_equal(L.A.values(), v), k  # values bitwise: they drive later node-HEM ties
        if agg is None:
            assert L.agg is None
        else:
            assert np.array_equal(L.agg.fine_to_coarse, agg), k


def test_worked_example(sp):
    # acceptance.cpp:63-93: agg [0,0,1,2,1,2], A_c = [[4,2,0],[2,12,1],[0,1,12]], nnz 7
    h = sp.Hierarchy(example_6x6(sp), sp.SolverConfig(coarse_target=3, max_levels=2))
    assert h.nlevels() == 2
    assert h.level(0).agg.fine_to_coarse.tolist() == [0, 0, 1, 2, 1, 2]
    Ac = h.level(1).A
    assert Ac.nnz() == 7
    assert np.array_equal(Ac.to_dense(), [[4, 2, 0], [2, 12, 1], [0, 1, 12]])
    P = h.level(0).P_to_coarser
    assert P.nrows() == 6 and P.ncols() == 3 and P.col_idx().tolist() == [0, 0, 1, 2, 1, 2]
    st = sp.stats(h)  # test_hierarchy.cpp:23-49: opc 25/18, gc 1.5
    assert st.operator_complexity == pytest.approx(25 / 18) and st.grid_complexity == 1.5


def test_hierarchy_shapes(sp):
    # test_hierarchy.cpp:60-68: 32^2, max_levels 3 -> 1024/512/256
    h = sp.Hierarchy(sp.poisson2d(32, 32), sp.SolverConfig(max_levels=3, coarse_target=1))
    assert [l.A.nrows() for l in h.levels()] == [1024, 512, 256]


def test_generators_match_reference(sp, ref):
    for args in [(16, 16, 0.0, 0.0, 0.0), (17, 23, 1.0, 100.0, 1.0), (9, 5, -2.0, 3.0, 0.5)]:
        A = sp.convdiff2d(*args)
        rp, ci, v = ref.convdiff2d(*args).arrays()
        assert np.array_equal(A.row_ptr(), rp) and np.array_equal(A.col_idx(), ci)
        assert np.array_equal(A.values(), v)


def test_rhs_random_matches_std_mt19937():
    # inc/problems.hpp:69-75; first draws of mt19937(42) through generate_canonical
    from paper_2007_00056_b200 import sparsh as sp
    r = sp.rhs_random(4, 42)
    assert np.all((r >= 0) & (r < 1)) and len(set(r)) == 4
    assert np.array_equal(sp.rhs_random(100, 42), sp.rhs_random(100, 42))


@pytest.mark.parametrize("mk", [
    lambda sp: sp.poisson2d(64, 64), lambda sp: sp.poisson3d(24), lambda sp: sp.aniso3d(20),
    lambda sp: sp.convdiff3d(14, 14, 14, 1.0, 100.0, 1.0, 1.0), lambda sp: sp.poisson3d_27(12),
    lambda sp: sp.convdiff2d(40, 40, 1.0, 100.0, 1.0)])
def test_hierarchy_bitexact_vs_oracle(sp, oracle_best, mk):
    A = mk(sp)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40, coarse_target=500))
    _same_hierarchy(h, oracle_best.hierarchy(A, 500, 40))


@pytest.mark.parametrize("seed", range(6))
def test_hierarchy_bitexact_random(sp, oracle_best, seed):
    A = (random_spd if seed % 2 else random_sparse)(sp, 60 + 7 * seed, seed, 0.15)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40, coarse_target=4))
    _same_hierarchy(h, oracle_best.hierarchy(A, 4, 40))


def test_galerkin_parallel_rows_bitexact(sp, port):
    # n_coarse >= 65536 takes the multithreaded Galerkin path; rows must still
    # accumulate in the reference's order (aggregation.hpp:118-150)
    A = sp.poisson3d(64)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=3, coarse_target=1000), _coarse_solver=-1)
    for k in range(2):
        L, C = h.level(k), h.level(k + 1).A
        agg, nc = port.node_hem(L.A)
        assert np.array_equal(L.agg.fine_to_coarse, agg) and nc >= 65536
        rp, ci, v = port.galerkin(L.A, agg, nc)
        assert np.array_equal(C.row_ptr(), rp) and np.array_equal(C.col_idx(), ci)
        assert np.array_equal(C.values(), v)


def test_node_hem_matches_oracle(sp, port):
    for n in (50, 80):
        A = random_spd(sp, n, n)
        agg, nc = port.node_hem(A)
        h = sp.Hierarchy(A, sp.SolverConfig(max_levels=2, coarse_target=1))
        if h.nlevels() > 1:
            assert np.array_equal(h.level(0).agg.fine_to_coarse, agg)
            assert h.level(0).agg.n_coarse == nc


def test_bad_inputs_raise_like_reference(sp):
    with pytest.raises(sp.InvalidArgument, match="columns not strictly increasing in row 0"):
        sp.CsrMatrix(2, 2, [0, 2, 3], [1, 0, 1], [1.0, 1.0, 1.0])
    with pytest.raises(sp.InvalidArgument, match="row_ptr"):
        sp.CsrMatrix(2, 2, [0, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(sp.InvalidArgument, match="must be square"):
        sp.Hierarchy(sp.CsrMatrix.from_triplets(2, 3, [(0, 0, 1.0)]))
    with pytest.raises(sp.InvalidArgument, match="coarse_target"):
        sp.Hierarchy(sp.poisson2d(4, 4), sp.SolverConfig(coarse_target=0))
    with pytest.raises(sp.InvalidArgument, match="Jacobi weight"):
        sp.SmootherKind.weighted_jacobi(1.5)
    with pytest.raises(sp.InvalidArgument, match="2000"):
        # default max_levels = 10 stops 1024^2 at 2048 rows: dense LU limit
        sp.Hierarchy(sp.poisson2d(64, 64), sp.SolverConfig(max_levels=1))


def test_setup_stencil27_matches_generated(sp):
    # sb_setup_stencil27 (generator fused into the setup, int64 offsets) builds
    # the same hierarchy as sb_gen_stencil27 + sb_setup
    cfg = sp.SolverConfig(max_levels=40)
    ha = sp.Hierarchy(sp._gen(sp._lib.lib().sb_gen_stencil27, 9, 10, 11, 26.0, -1.0), cfg)
    hb = sp.Hierarchy.from_stencil27(9, 10, 11, 26.0, -1.0, cfg)
    assert ha.nlevels() == hb.nlevels()
    for k in range(ha.nlevels()):
        a, b = ha.level(k), hb.level(k)
        assert a.A == b.A
        if a.agg is not None:
            assert np.array_equal(a.agg.fine_to_coarse, b.agg.fine_to_coarse)


@pytest.mark.parametrize("n", [16, 33, 48])
def test_setup_stencil27_equals_gen_plus_setup(sp, n):
    """sb_setup_stencil27 (operator generated straight into the setup, int64
    offsets: the C5 path) builds the same hierarchy as sb_gen_stencil27 +
    sb_setup, bit for bit (level CSRs and aggregates)."""
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
    a = sp.Hierarchy.from_stencil27(n, n, n, 26.0, -1.0, cfg)
    b = sp.Hierarchy(sp.poisson3d_27(n), cfg)
    la, lb = a.levels(), b.levels()
    assert len(la) == len(lb)
    for k, (x, y) in enumerate(zip(la, lb)):
        assert np.array_equal(np.asarray(x.A.row_ptr(), dtype=np.int64), np.asarray(y.A.row_ptr(), dtype=np.int64)), k
        assert np.array_equal(x.A.col_idx(), y.A.col_idx()), k
        assert np.array_equal(np.asarray(x.A.values()).view(np.uint64), np.asarray(y.A.values()).view(np.uint64)), k
        if y.agg is not None:
            assert np.array_equal(x.agg.fine_to_coarse, y.agg.fine_to_coarse), k
