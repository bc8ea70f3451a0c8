"""Time the C2 L0 Jacobi sweep / SpMV / V-cycle / whole solve for each library
variant under _variants/ (built by tools/build_variants.sh). GPU box only."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import ctypes as C, json, os, sys
sys.path.insert(0, %r)
import numpy as np, torch
from paper_2007_00056_b200 import sparsh as sp, _lib
wl = os.environ.get("VB_WL", "C2")
A = {"C2": lambda: sp.poisson3d(128), "C1": lambda: sp.poisson2d(1024, 1024), "C3": lambda: sp.aniso3d(256), "C4": lambda: sp.convdiff3d(256, 256, 256, 1.0, 100.0, 1.0, 1.0), "P27": lambda: sp.poisson3d_27(128), "P27_256": lambda: sp.poisson3d_27(256)}[wl]()
cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40)
h = sp.Hierarchy(A, cfg); ctx = h.ctx(); L = _lib.lib()
cp = sp.CycleParams.from_config(cfg)._abi()
out = {}
for kind, name, reps in [(0, "jac", 50), (1, "spmv", 50), (3, "vc", 10), (4, "vcg", 10)]:
    avg, cnt = C.c_double(), C.c_int()
    _lib.check(L.sb_time_kernel(ctx, kind, 0, C.byref(cp), reps, C.byref(avg), C.byref(cnt)))
    out[name] = round(avg.value * 1e3, 2)
n = A.nrows(); b = torch.ones(n, dtype=torch.float64, device="cuda"); x = torch.zeros_like(b)
tol = 1e-8 * float(np.sqrt(n)); rep = _lib.sb_report(); ts = []
for i in range(8):
    fn = L.sb_pbicgstab_dev if wl == "C4" else L.sb_pcg_dev
    _lib.check(fn(ctx, C.byref(cp), C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), tol, 1000, C.byref(rep)))
    if i >= 3: ts.append(L.sb_last_solve_ms(ctx))
out["solve_ms"] = round(sum(ts) / len(ts), 3); out["it"] = rep.iterations
print("RESULT " + json.dumps(out))
''' % ROOT

names = sys.argv[1:] or sorted(os.listdir(os.path.join(ROOT, "_variants")))
for nm in names:
    env = dict(os.environ)
    lib = os.path.join(ROOT, "_variants", nm, "libsparsh_b200.so")
    if nm != "base":
        env["SB_LIB"] = lib
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
    print(f"{nm:24s} {line[0][7:] if line else r.stderr[-400:]}", flush=True)
