"""Host setup time with the Galerkin products on the host (threads) vs the GPU."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00056_b200 import sparsh as sp  # noqa

gens = {"C2": lambda: sp.poisson3d(128), "C3": lambda: sp.aniso3d(256, 1e-3), "P27": lambda: sp.poisson3d_27(128)}
for wl in sys.argv[1:] or ["C2"]:
    A = gens[wl]()
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
    for gpu in (False, True, False, True):
        t0 = time.perf_counter()
        h = sp.Hierarchy(A, cfg, galerkin_gpu=gpu)
        dt = time.perf_counter() - t0
        print(f"{wl} galerkin_gpu={gpu}: setup {dt:.3f} s, {h.nlevels()} levels", flush=True)
        del h
