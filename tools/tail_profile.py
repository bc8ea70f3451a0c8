"""Eager V-cycles (sb_time_kernel kind 3: every kernel a separate launch, the
cluster tail included) of a workload, for ncu captures of k_tail."""
import ctypes as C
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00056_b200 import sparsh as sp, _lib  # noqa
wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
A = {"C2": lambda: sp.poisson3d(128), "T256": lambda: sp.poisson3d(256)}[wl]()
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg)
cp = sp.CycleParams.from_config(cfg)._abi()
ms, n = C.c_double(), C.c_int()
_lib.check(_lib.lib().sb_time_kernel(h.ctx(), 3, 0, C.byref(cp), 4, C.byref(ms), C.byref(n)))
print("eager vcycle ms", ms.value, "kernels", n.value)
