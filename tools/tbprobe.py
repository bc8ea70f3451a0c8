import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2007_00056_b200 import sparsh as sp
A = sp.aniso3d(20, 1e-3)
h = sp.Hierarchy(A, sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40))
x = np.random.default_rng(0).uniform(-1, 1, A.nrows()); f = x.copy()
out = h.smooth(0, sp.SmootherKind.weighted_jacobi(), x, f, 2)
print("ok", out[:3])
