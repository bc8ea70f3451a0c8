"""Real (graph-replayed) cost of the V-cycle below each level, tail on/off, plus
the tail kernel's per-phase timestamps. Run on the GPU box."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa
from paper_2007_00056_b200 import sparsh as sp, _lib  # noqa

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
A = {"C2": lambda: sp.poisson3d(128), "T256": lambda: sp.poisson3d(256), "P27_256": lambda: sp.poisson3d_27(256), "C1": lambda: sp.poisson2d(1024, 1024), "C3": lambda: sp.aniso3d(256),
     "G128": lambda: sp.graph_laplacian3d(128, seed=7)}[wl]()
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
L = _lib.lib()
cp = sp.CycleParams.from_config(cfg)._abi()
res = {}
for spec in sys.argv[2:] or ["0:1", "1048576:1"]:
    T, pdl = (spec.split(":") + ["1"])[:2]
    os.environ["SB_TAIL_ROWS"] = T
    os.environ["SB_PDL"] = pdl
    if os.environ.get("LC_TRACE") == "1":
        os.environ["SB_TAIL_TRACE"] = "1"
    h = sp.Hierarchy(A, cfg)
    ctx = h.ctx()
    tf, ct, smb = C.c_int(), C.c_int(), C.c_int()
    L.sb_tail_info(ctx, C.byref(tf), C.byref(ct), C.byref(smb))
    row = []
    for k in range(h.nlevels()):
        ms, n = C.c_double(), C.c_int()
        _lib.check(L.sb_time_kernel(ctx, 4, k, C.byref(cp), 50, C.byref(ms), C.byref(n)))
        row.append((k, h.level(k).A.nrows(), ms.value * 1e3, n.value))
    print(f"SB_TAIL_ROWS={T} SB_PDL={pdl}: tail_from={tf.value} ctas={ct.value} smem={smb.value}")
    for k, n, us, nk in row:
        print(f"   from L{k:2d} (n={n:8d}): {us:8.1f} us  {nk:3d} kernels")
    buf = (C.c_ulonglong * 256)()
    m = L.sb_tail_trace(ctx, buf, 256)
    if m > 1:
        t = np.array(buf[:m], dtype=np.float64)
        d = np.diff(t) / 1e3
        print(f"   tail phases: {m - 1}, total {(t[-1] - t[0]) / 1e3:.1f} us; first (load) {d[0]:.2f} us; "
              f"median {np.median(d[1:]):.2f} us; max {d[1:].max():.2f}")
        print("   ", " ".join(f"{x:.2f}" for x in d[:40]))
    del h
