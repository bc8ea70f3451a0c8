"""Phase stamps of k_crosspair inside a graph of 32 chained sweeps (needs the
SB_XP_TRACE variant: tools/build_variants.sh xptrace -DSB_XP_TRACE; SB_LIB=...).
Per sweep: launch-to-wait (prologue), wait release after the previous sweep's
last CTA exit, body (wait -> last exit).   python tools/xp_trace.py C2 6"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00056_b200 import sparsh as sp, _lib  # noqa

wl, k = sys.argv[1], int(sys.argv[2])
A = {"C2": lambda: sp.poisson3d(128), "T256": lambda: sp.poisson3d(256)}[wl]()
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg)
ctx = h.ctx()
L = _lib.lib()
L.sb_debug_xp_trace.argtypes = [C.c_void_p, C.c_int, C.c_int]
cp = sp.CycleParams.from_config(cfg)._abi()
ms, nl = C.c_double(), C.c_int()
_lib.check(L.sb_time_kernel(ctx, 5, k, C.byref(cp), 1, C.byref(ms), C.byref(nl)))
buf = np.zeros(6 * 65536, dtype=np.uint64)
L.sb_debug_xp_trace(buf.ctypes.data, 65536, 1)
_lib.check(L.sb_time_kernel(ctx, 5, k, C.byref(cp), 1, C.byref(ms), C.byref(nl)))
n = L.sb_debug_xp_trace(buf.ctypes.data, 65536, 1)
t = buf[:6 * n].reshape(n, 6).astype(np.int64)
print("per sweep (graph):", ms.value * 1e3 / nl.value, "us;", n, "CTA records")
t = t[np.argsort(t[:, 1])]
G = int(t[:, 3].max()) + 1
S = n // G
sw = [t[i * G:(i + 1) * G] for i in range(S)]
rows = []
for i in range(1, S):
    a, b = sw[i - 1], sw[i]
    rows.append((b[:, 1].min() - a[:, 2].max(), b[:, 2].max() - b[:, 1].min(), b[:, 1].min() - b[:, 0].min(),
                 b[:, 2].max() - a[:, 2].max(), np.median(b[:, 2] - b[:, 1])))
r = np.array(rows, dtype=float)
ld = t[:, 4]
okl = ld > 0
print("per-CTA median ns: wait -> loads done %.0f | loads -> last thread done %.0f | done -> trace %.0f" % (
    np.median(ld[okl] - t[okl, 1]), np.median(t[okl, 2] - ld[okl]), np.median(t[:, 5] - t[:, 2])))
print("median ns: wait-release after prev exit %.0f | body (first wait -> last exit) %.0f | entry -> wait %.0f |"
      " exit-to-exit %.0f | per-CTA body %.0f" % tuple(np.median(r, axis=0)))
