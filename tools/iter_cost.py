"""Per-iteration cost of the T256 PCG graph: solves stopped at 8 / 16 / 32
iterations (tol tiny), device time per solve, and the standalone V-cycle graph
(cold L2) for comparison."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00056_b200 import sparsh as sp, _lib  # noqa

A = sp.poisson3d(256)
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg)
ctx = h.ctx()
L = _lib.lib()
cp = sp.CycleParams.from_config(cfg)._abi()
n = A.nrows()
b = torch.ones(n, dtype=torch.float64, device="cuda")
x = torch.zeros(n, dtype=torch.float64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
rep = _lib.sb_report()
res = {}
for k in (8, 16, 32):
    t = []
    for r in range(6):
        flush.zero_()
        torch.cuda.synchronize()
        _lib.check(L.sb_pcg_dev(ctx, C.byref(cp), C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), 1e-300, k,
                                C.byref(rep)))
        if r >= 2:
            t.append(L.sb_last_solve_ms(ctx))
    res[k] = np.mean(t)
    print(k, "iterations:", round(res[k], 3), "ms", rep.iterations)
print("per iteration (16 -> 32):", round((res[32] - res[16]) / 16, 4), "ms; (8 -> 16):", round((res[16] - res[8]) / 8, 4))
ms, nl = C.c_double(), C.c_int()
_lib.check(L.sb_time_kernel_cold(ctx, 4, 0, C.byref(cp), 5, 512 << 20, C.byref(ms), C.byref(nl)))
print("V-cycle graph (cold L2):", round(ms.value, 4), "ms")
_lib.check(L.sb_time_kernel(ctx, 4, 0, C.byref(cp), 10, C.byref(ms), C.byref(nl)))
print("V-cycle graph (back to back):", round(ms.value, 4), "ms")
