"""Eager-launch PCG (the partitioned path with one virtual rank) inside NVTX
range 'prof', for an ncu launch list of one whole solve (graph launches with
conditional nodes cannot be profiled per kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa
import torch  # noqa
from paper_2007_00056_b200 import sparsh as sp  # noqa
from paper_2007_00056_b200.dist import DistSolver  # noqa

A = sp.poisson3d(128)
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg)
ds = DistSolver(h, 1, 131072)
b = sp.rhs_ones(A.nrows())
cp = sp.CycleParams.from_config(cfg)
tol = 1e-8 * float(np.linalg.norm(b))
r = ds.pcg(b, cp, tol, 1000)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
r = ds.pcg(b, cp, tol, 1000)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("iterations", r.report.iterations, "ms", ds.last_solve_ms())
