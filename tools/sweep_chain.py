"""In-graph cost of one Jacobi sweep per level (kind 5: 32 chained sweeps as one
graph) beside the isolated back-to-back launch time (kind 0).
  python tools/sweep_chain.py C2"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00056_b200 import sparsh as sp, _lib  # noqa

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
A = {"C2": lambda: sp.poisson3d(128), "T256": lambda: sp.poisson3d(256), "C1": lambda: sp.poisson2d(1024, 1024),
     "P27": lambda: sp.poisson3d_27(128), "P27_256": lambda: sp.poisson3d_27(256), "G128": lambda: sp.graph_laplacian3d(128, seed=7)}[wl]()
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg)
ctx = h.ctx()
L = _lib.lib()
cp = sp.CycleParams.from_config(cfg)._abi()
for k, lv in enumerate(h.levels()[:-1]):
    ms, nl = C.c_double(), C.c_int()
    _lib.check(L.sb_time_kernel(ctx, 5, k, C.byref(cp), 20, C.byref(ms), C.byref(nl)))
    chain = ms.value * 1e3 / nl.value
    _lib.check(L.sb_time_kernel(ctx, 0, k, C.byref(cp), 50, C.byref(ms), C.byref(nl)))
    print(f"L{k:2d} n={lv.A.nrows():9d}  in-graph sweep {chain:7.2f} us   stream launch {ms.value * 1e3:7.2f} us")
