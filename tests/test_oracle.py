"""Pins the plain-C oracle restatement (oracle/sparsh_oracle.c) against the
reference's own outputs: the committed golden fixtures (made by
tests/golden/make_golden.py from oracle/_ref) and, where the reference build is
present, the reference itself on fresh inputs. CPU only."""
import glob
import os

import numpy as np
import pytest

from conftest import golden_path
from helpers import example_6x6, from_npz

CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(golden_path("*.npz"))
               if not p.endswith("example_6x6.npz") and not os.path.basename(p).startswith("config_"))


def test_example_6x6_known_answer(sp, port):
    # acceptance.cpp:63-93 / SPEC.md:51: agg [0,0,1,2,1,2], A*1 = (3,3,8,7,7,6)
    A = example_6x6(sp)
    agg, nc = port.node_hem(A)
    assert agg.tolist() == [0, 0, 1, 2, 1, 2] and nc == 3
    assert port.spmv(A, np.ones(6)).tolist() == [3, 3, 8, 7, 7, 6]
    g = np.load(golden_path("example_6x6.npz"))
    assert np.array_equal(g["agg"], agg) and np.array_equal(g["spmv_ones"], port.spmv(A, np.ones(6)))


@pytest.mark.parametrize("name", CASES)
def test_port_matches_reference_golden(sp, port, name):
    d = np.load(golden_path(f"{name}.npz"))
    A = from_npz(sp, d)
    assert np.array_equal(port.spmv(A, d["f"]), d["spmv_f"])
    assert np.array_equal(port.jacobi(A, 2.0 / 3.0, d["f"], d["b"], 3), d["jacobi3"])
    h = port.hierarchy(A, 100, 40)
    assert h.nlevels() == int(d["nlevels"])
    for k in range(h.nlevels()):
        rp, ci, v, agg = h.level(k)
        assert np.array_equal(rp, d[f"L{k}_rp"]) and np.array_equal(ci, d[f"L{k}_ci"])
        assert np.array_equal(v, d[f"L{k}_v"])
        if agg is not None:
            assert np.array_equal(agg, d[f"L{k}_agg"])
    assert np.array_equal(h.vcycle(d["b"], np.zeros(A.nrows())), d["vcycle"])
    res = getattr(h, str(d["solver"]))(d["b"], float(d["tol"]), 500)
    assert res.iterations == int(d["iters"]) and res.termination == int(d["term"])
    assert np.array_equal(res.x, d["x"])
    assert np.array_equal(np.array(res.residual_history), d["hist"])
    assert res.true_residual == float(d["true_res"])
    amg = h.amg_solve(d["b"], float(d["tol"]), 40)
    assert amg.iterations == int(d["amg_iters"]) and np.array_equal(amg.x, d["amg_x"])


@pytest.mark.parametrize("mk", [
    lambda sp: sp.poisson3d(20), lambda sp: sp.aniso3d(16), lambda sp: sp.poisson2d(48, 40),
    lambda sp: sp.convdiff3d(12, 12, 12, 1.0, 100.0, 1.0, 1.0), lambda sp: sp.poisson3d_27(10)])
def test_port_matches_reference_live(sp, port, ref, mk):
    A = mk(sp)
    b = sp.rhs_random(A.nrows(), 42)
    rh, ph = ref.hierarchy(A, 500, 40), port.hierarchy(A, 500, 40)
    assert rh.nlevels() == ph.nlevels()
    for k in range(rh.nlevels()):
        for a, c in zip(rh.level(k), ph.level(k)):
            assert (a is None and c is None) or np.array_equal(a, c)
    assert np.array_equal(rh.vcycle(b, np.zeros(A.nrows())), ph.vcycle(b, np.zeros(A.nrows())))
    tol = 1e-8 * np.linalg.norm(b)
    for solver in ("pcg", "pbicgstab"):
        r1, r2 = getattr(rh, solver)(b, tol, 100), getattr(ph, solver)(b, tol, 100)
        assert r1.iterations == r2.iterations and np.array_equal(r1.x, r2.x)
        assert r1.residual_history == r2.residual_history
    a1, a2 = rh.amg_solve(b, tol, 30), ph.amg_solve(b, tol, 30)
    assert a1.iterations == a2.iterations and np.array_equal(a1.x, a2.x)


def test_port_identity_cg_and_breakdowns(sp, port, ref):
    # test_krylov.cpp:78-85 (pAp = 0 breakdown), :106-112 (zero rhs)
    A = sp.CsrMatrix.from_triplets(2, 2, [(0, 0, 1.0), (1, 1, -1.0)])
    for o in (port, ref):
        h = o.hierarchy(A, 500, 40)
        r = h.pcg(np.array([1.0, 1.0]), 1e-10, 10, amg=False)
        assert r.termination == 2 and r.iterations == 0
    A = sp.poisson2d(4, 4)
    for o in (port, ref):
        r = o.hierarchy(A, 500, 40).pcg(np.zeros(16), 1e-8, 10)
        assert r.termination == 0 and r.iterations == 0 and not r.x.any()


def test_amg_divergence_reported(sp, port, ref):
    # test_cycle.cpp:135-148 analogue with Jacobi: [[1,3],[3,1]] diverges
    A = sp.CsrMatrix.from_dense([[1.0, 3.0], [3.0, 1.0]])
    p = port.hierarchy(A, 1, 40)
    r = ref.hierarchy(A, 1, 40)
    a, b = p.amg_solve(np.array([1.0, -1.0]), 1e-8, 50), r.amg_solve(np.array([1.0, -1.0]), 1e-8, 50)
    assert a.status == 2 and b.status == 2 and "diverged" in b.error


def test_reference_generators_match_product(sp, ref):
    """The reference-built 3D generators (oracle/ref_capi.cpp, used by bench.py's
    reference arm and the config fixtures) and the product's (sb_gen_*) give the
    same CSR bit for bit."""
    import oracle as orc

    def same(rm, A):
        rp, ci, v = rm.arrays()
        return (np.array_equal(rp, A.row_ptr()) and np.array_equal(ci, A.col_idx())
                and np.array_equal(v.view(np.uint64), np.asarray(A.values()).view(np.uint64)))

    assert same(ref.poisson3d(9), sp.poisson3d(9))
    assert same(ref.aniso3d(8, 1e-3), sp.aniso3d(8, 1e-3))
    assert same(ref.convdiff3d(7, 8, 9, 1.0, 100.0, 1.0, 1.0), sp.convdiff3d(7, 8, 9, 1.0, 100.0, 1.0, 1.0))
    assert same(ref.stencil27(6, 6, 6), sp.poisson3d_27(6))
    assert same(ref.convdiff2d(12, 10, 0.0, 0.0, 0.0), sp.poisson2d(12, 10))
    rp, ci, v = orc.graph_laplacian3d_arrays(9, seed=7)
    G = sp.graph_laplacian3d(9, seed=7)
    assert np.array_equal(rp, G.row_ptr()) and np.array_equal(ci, G.col_idx())
    assert np.array_equal(v.view(np.uint64), np.asarray(G.values()).view(np.uint64))


def test_config_fixtures_consistent():
    """tests/golden/config_*.npz (the reference at the BASELINE configs) hold the
    survey-measured iteration counts and converged."""
    import json
    expect = {"C1": 60, "C2": 22, "C3": 43, "P27_128": 20}
    for name, k in expect.items():
        p = golden_path(f"config_{name}.npz")
        if not os.path.exists(p):
            continue
        m = json.loads(str(np.load(p)["meta"]))
        assert m["iterations"] == k and m["termination"] == 0, (name, m["iterations"])
