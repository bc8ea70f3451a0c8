"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, the
unmodified sparsh headers compiled by oracle/Makefile). Run in the build
container (needs /root/reference):  python tests/golden/make_golden.py

Each fixture pins the plain-C oracle restatement and the GPU path to the
reference's own outputs on small inputs (SURVEY.md §8c known answers +
recorded trajectories)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

from paper_2007_00056_b200 import sparsh as sp  # noqa: E402  (generators + CsrMatrix only)
import oracle as orc  # noqa: E402


def example_6x6():
    """tests/oracles.hpp:53-62 (the paper's worked example)."""
    return sp.CsrMatrix.from_dense([[4, -2, 0, 0, 1, 0], [-2, 4, 1, 0, 0, 0], [0, 1, 4, 1, 2, 0],
                                    [0, 0, 1, 4, 0, 2], [1, 0, 2, 0, 4, 0], [0, 0, 0, 2, 0, 4]])


CASES = {
    # name: (matrix builder, solver, rhs)
    "poisson2d_16": (lambda: sp.poisson2d(16, 16), "pcg", "ones"),
    "poisson2d_32_rand": (lambda: sp.poisson2d(32, 32), "pcg", "random"),
    "poisson3d_12": (lambda: sp.poisson3d(12), "pcg", "ones"),
    "aniso3d_12": (lambda: sp.aniso3d(12, 1e-3), "pcg", "ones"),
    "convdiff2d_24": (lambda: sp.convdiff2d(24, 24, 1.0, 100.0, 1.0), "pbicgstab", "ones"),
    "convdiff3d_10": (lambda: sp.convdiff3d(10, 10, 10, 1.0, 100.0, 1.0, 1.0), "pbicgstab", "random"),
    "poisson27_8": (lambda: sp.poisson3d_27(8), "pcg", "ones"),
}


def main():
    R = orc.Ref()
    # known answer: 6x6 example
    A = example_6x6()
    m = R.matrix(A)
    agg, nc = m.node_hem()
    y = m.spmv(np.ones(6))
    np.savez(os.path.join(HERE, "example_6x6.npz"), rp=A.row_ptr(), ci=A.col_idx(), v=A.values(),
             agg=agg, nc=nc, spmv_ones=y)
    for name, (mk, solver, rhs) in CASES.items():
        A = mk()
        n = A.nrows()
        b = sp.rhs_ones(n) if rhs == "ones" else sp.rhs_random(n, 42)
        h = R.hierarchy(A, 100, 40)
        lv = {}
        for k in range(h.nlevels()):
            rp, ci, v, ag = h.level(k)
            lv[f"L{k}_rp"], lv[f"L{k}_ci"], lv[f"L{k}_v"] = rp, ci, v
            if ag is not None:
                lv[f"L{k}_agg"] = ag
        x0 = np.zeros(n)
        vc = h.vcycle(b, x0)
        f = sp.rhs_random(n, 7)
        ax = R.matrix(A).spmv(f)
        jac = R.matrix(A).smooth(0, 2.0 / 3.0, f, b, 3)
        tol = 1e-8 * float(np.linalg.norm(b))
        res = getattr(h, solver)(b, tol, 500)
        amg = h.amg_solve(b, tol, 40)
        np.savez(os.path.join(HERE, f"{name}.npz"), rp=A.row_ptr(), ci=A.col_idx(), v=A.values(), b=b,
                 nlevels=h.nlevels(), vcycle=vc, f=f, spmv_f=ax, jacobi3=jac, solver=solver, tol=tol,
                 iters=res.iterations, term=res.termination, x=res.x,
                 hist=np.array(res.residual_history), true_res=res.true_residual,
                 amg_iters=amg.iterations, amg_x=amg.x, amg_hist=np.array(amg.residual_history), **lv)
        print(name, n, h.nlevels(), solver, res.iterations, amg.iterations)


if __name__ == "__main__":
    main()
