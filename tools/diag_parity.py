"""Diagnostic: where do GPU-vs-reference differences come from? Compares one
V-cycle and same-iteration-count Krylov solutions with the inverse-GEMV coarse
solve vs the bit-exact LU substitution, and with the identity preconditioner."""
import glob
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
from paper_2007_00056_b200 import sparsh as sp  # noqa
import oracle as orc  # noqa
from helpers import from_npz, rel  # noqa

P = orc.Port()
cfgj = dict(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
for path in sorted(glob.glob(os.path.join(ROOT, "tests/golden/*.npz"))):
    if "example" in path:
        continue
    d = np.load(path)
    A = from_npz(sp, d)
    solver = str(d["solver"])
    k = int(d["iters"])
    cp = sp.CycleParams(6, 6, sp.SmootherKind.weighted_jacobi())
    out = [os.path.basename(path), solver, k]
    for exact in (False, True):
        h = sp.Hierarchy(A, sp.SolverConfig(coarse_target=100, **cfgj), coarse_exact=exact)
        M = sp.make_amg_preconditioner(h, cp)
        vc = rel(sp.vcycle(h, 0, d["b"], np.zeros(A.nrows()), cp), d["vcycle"])
        x = getattr(sp, solver)(A, d["b"], M, 1e-300, k).x
        out += [f"exact={int(exact)} vc={vc:.1e} x={rel(x, d['x']):.1e}"]
    o = P.hierarchy(A, 100, 40)
    xi = getattr(sp, solver)(A, d["b"], sp.Preconditioner.identity(), 1e-300, 6).x
    xo = getattr(o, solver)(d["b"], 1e-300, 6, amg=False).x
    out += [f"identity(6 it) x={rel(xi, xo):.1e}"]
    print(*out)
