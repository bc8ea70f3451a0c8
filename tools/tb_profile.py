"""Two fused sweeps (k_cross_tb2) on level 0 of a workload, for ncu captures."""
import sys
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa
from paper_2007_00056_b200 import sparsh as sp  # noqa
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = sp.poisson3d(n)
h = sp.Hierarchy(A, sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40))
x = np.random.default_rng(0).uniform(-1, 1, A.nrows())
for _ in range(3):
    h.smooth(0, sp.SmootherKind.weighted_jacobi(), x, x, 2)
print("done")
