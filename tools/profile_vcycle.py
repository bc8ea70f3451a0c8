"""Profiling target (run under ncu on the GPU box): builds a config's hierarchy,
warms up, then runs ONE V-cycle and ONE PCG solve inside NVTX range 'prof'.
  ncu --nvtx --nvtx-include 'prof/' --metrics gpu__time_duration.sum --csv python tools/profile_vcycle.py C2
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa
import torch  # noqa
from paper_2007_00056_b200 import sparsh as sp, _lib  # noqa

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
what = sys.argv[2] if len(sys.argv) > 2 else "both"
gen = {"C2": lambda: sp.poisson3d(128), "C1": lambda: sp.poisson2d(1024, 1024),
       "C3": lambda: sp.aniso3d(256), "M64": lambda: sp.poisson3d(64), "T256": lambda: sp.poisson3d(256),
       "C4": lambda: sp.convdiff3d(256, 256, 256, 1.0, 100.0, 1.0, 1.0), "P27": lambda: sp.poisson3d_27(128),
       "P27_256": lambda: sp.poisson3d_27(256),
       "G128": lambda: sp.graph_laplacian3d(128, seed=7)}[wl]
A = gen()
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg)
ctx = h.ctx()
L = _lib.lib()
cp = sp.CycleParams.from_config(cfg)._abi()
n = A.nrows()
b = torch.ones(n, dtype=torch.float64, device="cuda")
x = torch.zeros(n, dtype=torch.float64, device="cuda")
tol = 1e-8 * float(np.sqrt(n))
rep = _lib.sb_report()
for _ in range(2):
    _lib.check(L.sb_vcycle_dev(ctx, C.byref(cp), 0, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), 1))
    _lib.check(L.sb_pcg_dev(ctx, C.byref(cp), C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), tol, 1000,
                            C.byref(rep)))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
if what in ("both", "vcycle"):
    _lib.check(L.sb_vcycle_dev(ctx, C.byref(cp), 0, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), 1))
if what in ("both", "solve"):
    _lib.check(L.sb_pcg_dev(ctx, C.byref(cp), C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), tol, 1000,
                            C.byref(rep)))
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("levels", [(l.A.nrows(), l.A.nnz()) for l in h.levels()])
print("iterations", rep.iterations, "solve ms", L.sb_last_solve_ms(ctx))
