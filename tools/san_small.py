import sys, numpy as np
sys.path.insert(0, '.')
from paper_2007_00056_b200 import sparsh as sp
A = sp.poisson3d(16)
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg)
x = h.spmv(0, np.ones(A.nrows()))
print("spmv ok")
b = sp.rhs_ones(A.nrows())
r = sp.pcg(A, b, sp.make_amg_preconditioner(h, sp.CycleParams.from_config(cfg)), 1e-8*np.linalg.norm(b), 100)
print(r.report.iterations)
