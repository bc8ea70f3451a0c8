"""Profiling target: one Jacobi sweep of level K of a workload's hierarchy
(sb_time_kernel kind 0, 2 launches: ncu --launch-skip 1 -c 1 picks the 2nd).
  ncu -k regex:k_csr_tile --launch-skip 1 -c 1 --set full python tools/prof_level.py G128 30"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00056_b200 import sparsh as sp, _lib  # noqa

wl, k = sys.argv[1], int(sys.argv[2])
A = {"G128": lambda: sp.graph_laplacian3d(128, seed=7), "C2": lambda: sp.poisson3d(128)}[wl]()
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg)
cp = sp.CycleParams.from_config(cfg)._abi()
ms, nl = C.c_double(), C.c_int()
_lib.check(_lib.lib().sb_time_kernel(h.ctx(), 0, k, C.byref(cp), 1, C.byref(ms), C.byref(nl)))
print("level", k, "sweep ms", ms.value)
