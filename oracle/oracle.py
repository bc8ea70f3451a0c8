"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracles.

Two oracles, same interface:
  * ``Port``: the plain-C restatement (oracle/sparsh_oracle.c ->
    oracle/_build/libsparsh_oracle.so);
  * ``Ref``:  the reference's own headers compiled behind oracle/ref_capi.cpp
    (oracle/_ref/libsparsh_ref.so; built only where /root/reference exists,
    but the .so travels to the GPU box).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libsparsh_oracle.so")
PORT_FMA_SO = os.path.join(HERE, "_build", "libsparsh_oracle_fma.so")
REF_SO = os.path.join(HERE, "_ref", "libsparsh_ref.so")
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int32)


def build(ref: bool = True) -> None:
    """make -C oracle (the restatement always; _ref only when the reference exists)."""
    targets = ["oracle"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/include") else [])
    subprocess.run(["make", "-C", HERE] + targets, check=True, capture_output=True)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("termination", C.c_int), ("wall_time", C.c_double),
                ("true_residual", C.c_double), ("hist_len", C.c_int), ("hist_cap", C.c_int),
                ("residual_history", _D), ("time_history", _D)]


class SolveOut:
    def __init__(self, x, rep: Report, hr, ht):
        m = min(rep.hist_len, rep.hist_cap)
        self.x = x
        self.iterations = rep.iterations
        self.termination = rep.termination
        self.wall_time = rep.wall_time
        self.true_residual = rep.true_residual
        self.residual_history = list(hr[:m])
        self.time_history = list(ht[:m])


def _new_report(cap):
    hr, ht = np.zeros(cap), np.zeros(cap)
    r = Report()
    r.hist_cap = cap
    r.residual_history = hr.ctypes.data_as(_D)
    r.time_history = ht.ctypes.data_as(_D)
    return r, hr, ht


# ---------------------------------------------------------------------------
# restatement (plain C)
# ---------------------------------------------------------------------------
class OcCsr(C.Structure):
    _fields_ = [("n", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("rp", _I), ("ci", _I), ("v", _D)]


class Port:
    """The restatement; fma=True loads the FMA-contracted build (noise-floor probe)."""
    kind = "port"

    def __init__(self, fma: bool = False):
        so = PORT_FMA_SO if fma else PORT_SO
        if not os.path.exists(so):
            build(ref=False)
        L = C.CDLL(so)
        L.oc_hier_build.restype = C.c_void_p
        L.oc_hier_build.argtypes = [C.POINTER(OcCsr), C.c_int32, C.c_int, C.POINTER(C.c_int)]
        L.oc_hier_free.argtypes = [C.c_void_p]
        L.oc_hier_nlevels.argtypes = [C.c_void_p]
        L.oc_hier_level.restype = C.POINTER(OcCsr)
        L.oc_hier_level.argtypes = [C.c_void_p, C.c_int]
        L.oc_hier_agg.restype = _I
        L.oc_hier_agg.argtypes = [C.c_void_p, C.c_int]
        L.oc_hier_set_cycle.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double]
        L.oc_vcycle.restype = C.c_int32
        L.oc_vcycle.argtypes = [C.c_void_p, C.c_int, _D, _D]
        L.oc_pcg.argtypes = [C.POINTER(OcCsr), C.c_void_p, _D, _D, C.c_double, C.c_int, C.POINTER(Report)]
        L.oc_pbicgstab.argtypes = L.oc_pcg.argtypes
        L.oc_amg_solve.restype = C.c_int
        L.oc_amg_solve.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int, C.POINTER(Report)]
        L.oc_spmv.argtypes = [C.POINTER(OcCsr), _D, _D]
        L.oc_residual.argtypes = [C.POINTER(OcCsr), _D, _D, _D]
        L.oc_jacobi.restype = C.c_int32
        L.oc_jacobi.argtypes = [C.POINTER(OcCsr), C.c_double, _D, _D, C.c_int]
        L.oc_node_hem.restype = C.c_int32
        L.oc_node_hem.argtypes = [C.POINTER(OcCsr), _I]
        L.oc_coarse_solve.argtypes = [C.c_void_p, _D, _D]
        L.oc_restrict.argtypes = [C.c_int32, _I, C.c_int32, _D, _D]
        L.oc_galerkin.argtypes = [C.POINTER(OcCsr), _I, C.c_int32, C.POINTER(OcCsr)]
        L.oc_prolong_add.argtypes = [C.c_int32, _I, _D, _D]
        L.oc_set_dot_mode.argtypes = [C.c_int]
        self.L = L

    def set_dot_mode(self, mode):
        """0: the reference's sequential dots; 1: reordered (blocked + pairwise) dots
        (noise-floor measurements only, tools/noise_floor.py)."""
        self.L.oc_set_dot_mode(int(mode))

    def _csr(self, rp, ci, v, n, ncols=None):
        rp = np.ascontiguousarray(rp, dtype=np.int32)
        ci = np.ascontiguousarray(ci, dtype=np.int32)
        v = _d(v)
        s = OcCsr(n, n if ncols is None else ncols, int(rp[-1]), rp.ctypes.data_as(_I),
                  ci.ctypes.data_as(_I), v.ctypes.data_as(_D))
        s._keep = (rp, ci, v)
        return s

    def spmv(self, A, x):
        s = self._csr(A.row_ptr(), A.col_idx(), A.values(), A.nrows(), A.ncols())
        x = _d(x)
        y = np.empty(A.nrows())
        self.L.oc_spmv(C.byref(s), x.ctypes.data_as(_D), y.ctypes.data_as(_D))
        return y

    def residual(self, A, x, f):
        s = self._csr(A.row_ptr(), A.col_idx(), A.values(), A.nrows(), A.ncols())
        x, f = _d(x), _d(f)
        r = np.empty(A.nrows())
        self.L.oc_residual(C.byref(s), x.ctypes.data_as(_D), f.ctypes.data_as(_D), r.ctypes.data_as(_D))
        return r

    def jacobi(self, A, omega, x, f, sweeps):
        s = self._csr(A.row_ptr(), A.col_idx(), A.values(), A.nrows(), A.ncols())
        x = _d(x).copy()
        f = _d(f)
        bad = self.L.oc_jacobi(C.byref(s), omega, x.ctypes.data_as(_D), f.ctypes.data_as(_D), sweeps)
        if bad >= 0:
            raise ValueError(f"smooth: zero diagonal entry in row {bad}")
        return x

    def node_hem(self, A):
        s = self._csr(A.row_ptr(), A.col_idx(), A.values(), A.nrows())
        out = np.empty(A.nrows(), dtype=np.int32)
        nc = self.L.oc_node_hem(C.byref(s), out.ctypes.data_as(_I))
        return out, int(nc)

    def hierarchy(self, A, coarse_target=500, max_levels=40):
        return PortHier(self, A, coarse_target, max_levels)

    def galerkin(self, A, agg, nc):
        s = self._csr(A.row_ptr(), A.col_idx(), A.values(), A.nrows())
        agg = np.ascontiguousarray(agg, dtype=np.int32)
        out = OcCsr()
        self.L.oc_galerkin(C.byref(s), agg.ctypes.data_as(_I), nc, C.byref(out))
        rp = np.ctypeslib.as_array(out.rp, shape=(nc + 1,)).copy()
        ci = np.ctypeslib.as_array(out.ci, shape=(out.nnz,)).copy()
        v = np.ctypeslib.as_array(out.v, shape=(out.nnz,)).copy()
        libc = C.CDLL(None)
        for p in (out.rp, out.ci, out.v):
            libc.free(C.cast(p, C.c_void_p))
        return rp, ci, v


class PortHier:
    def __init__(self, port: Port, A, coarse_target, max_levels):
        self.P = port
        self.A0 = port._csr(A.row_ptr(), A.col_idx(), A.values(), A.nrows())
        err = C.c_int(0)
        self.h = port.L.oc_hier_build(C.byref(self.A0), coarse_target, max_levels, C.byref(err))
        if not self.h:
            raise ValueError(f"oracle hierarchy build failed (code {err.value})")

    def __del__(self):
        if getattr(self, "h", None):
            self.P.L.oc_hier_free(self.h)
            self.h = None

    def nlevels(self):
        return self.P.L.oc_hier_nlevels(self.h)

    def level(self, k):
        s = self.P.L.oc_hier_level(self.h, k).contents
        n, nnz = s.n, s.nnz
        rp = np.ctypeslib.as_array(s.rp, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(s.ci, shape=(nnz,)).copy() if nnz else np.zeros(0, np.int32)
        v = np.ctypeslib.as_array(s.v, shape=(nnz,)).copy() if nnz else np.zeros(0)
        agg = None
        if k + 1 < self.nlevels():
            agg = np.ctypeslib.as_array(self.P.L.oc_hier_agg(self.h, k), shape=(n,)).copy()
        return rp, ci, v, agg

    def set_cycle(self, pre=6, post=6, omega=2.0 / 3.0):
        self.P.L.oc_hier_set_cycle(self.h, pre, post, omega)

    def vcycle(self, f, x, k=0):
        f, x = _d(f), _d(x).copy()
        self.P.L.oc_vcycle(self.h, k, f.ctypes.data_as(_D), x.ctypes.data_as(_D))
        return x

    def coarse_solve(self, f):
        f = _d(f)
        x = np.empty(f.size)
        self.P.L.oc_coarse_solve(self.h, f.ctypes.data_as(_D), x.ctypes.data_as(_D))
        return x

    def _krylov(self, fn, b, tol, max_iters, amg):
        b = _d(b)
        x = np.empty(b.size)
        rep, hr, ht = _new_report(max(max_iters, 0) + 2)
        fn(C.byref(self.A0), self.h if amg else None, b.ctypes.data_as(_D), x.ctypes.data_as(_D),
           tol, max_iters, C.byref(rep))
        return SolveOut(x, rep, hr, ht)

    def pcg(self, b, tol, max_iters, amg=True):
        return self._krylov(self.P.L.oc_pcg, b, tol, max_iters, amg)

    def pbicgstab(self, b, tol, max_iters, amg=True):
        return self._krylov(self.P.L.oc_pbicgstab, b, tol, max_iters, amg)

    def amg_solve(self, b, tol, max_cycles):
        b = _d(b)
        x = np.empty(b.size)
        rep, hr, ht = _new_report(max(max_cycles, 0) + 2)
        st = self.P.L.oc_amg_solve(self.h, b.ctypes.data_as(_D), x.ctypes.data_as(_D), tol, max_cycles,
                                   C.byref(rep))
        out = SolveOut(x, rep, hr, ht)
        out.status = st
        return out


# ---------------------------------------------------------------------------
# the reference itself (compiled headers behind ref_capi.cpp)
# ---------------------------------------------------------------------------
class Ref:
    kind = "reference"

    def __init__(self):
        if not os.path.exists(REF_SO):
            build(ref=True)
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        P = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_uint]
        L.ref_csr_new.argtypes = [C.c_int32, C.c_int32, _I, _I, _D, C.POINTER(P)]
        L.ref_convdiff2d.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.POINTER(P)]
        L.ref_stencil7.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, _D, C.POINTER(P)]
        L.ref_convdiff3d.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.POINTER(P)]
        L.ref_stencil27.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.POINTER(P)]
        L.ref_csr_free.argtypes = [P]
        L.ref_csr_info.argtypes = [P, _I, _I, C.POINTER(C.c_int64)]
        L.ref_csr_copy.argtypes = [P, _I, _I, _D]
        L.ref_spmv.argtypes = [P, _D, _D]
        L.ref_residual.argtypes = [P, _D, _D, _D]
        L.ref_smooth.argtypes = [P, C.c_int, C.c_double, _D, _D, C.c_int]
        L.ref_spmv_transpose.argtypes = [P, _D, _D]
        L.ref_node_hem.argtypes = [P, _I, _I]
        L.ref_hier_new.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(P)]
        L.ref_hier_free.argtypes = [P]
        L.ref_hier_nlevels.argtypes = [P]
        L.ref_hier_level_info.argtypes = [P, C.c_int, _I, C.POINTER(C.c_int64), _I]
        L.ref_hier_level_copy.argtypes = [P, C.c_int, _I, _I, _D, _I]
        L.ref_hier_level_matrix.restype = P
        L.ref_hier_level_matrix.argtypes = [P, C.c_int]
        L.ref_hier_set_cycle.argtypes = [P, C.c_int, C.c_double, C.c_int, C.c_int]
        L.ref_vcycle.argtypes = [P, C.c_int, _D, _D]
        L.ref_coarse_solve.argtypes = [P, _D, _D]
        L.ref_krylov.argtypes = [C.c_int, P, P, _D, _D, C.c_double, C.c_int, C.POINTER(Report)]
        L.ref_amg_solve.argtypes = [P, _D, _D, C.c_double, C.c_int, C.POINTER(Report)]
        L.ref_read_mm.argtypes = [C.c_char_p, C.POINTER(P)]
        L.ref_memory_plan.argtypes = [P, C.c_int, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                      C.POINTER(C.c_longlong)]
        L.ref_csr_bytes.restype = C.c_longlong
        L.ref_csr_bytes.argtypes = [P]
        L.ref_write_mm.argtypes = [P, C.c_char_p]
        self.L = L

    def check(self, rc):
        if rc == 0:
            return
        msg = self.L.ref_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)

    def set_threads(self, n):
        self.L.ref_set_threads(int(n))

    def matrix(self, A):
        rp = np.ascontiguousarray(A.row_ptr(), dtype=np.int32)
        h = C.c_void_p()
        self.check(self.L.ref_csr_new(A.nrows(), A.ncols(), rp.ctypes.data_as(_I),
                                      np.ascontiguousarray(A.col_idx()).ctypes.data_as(_I),
                                      _d(A.values()).ctypes.data_as(_D), C.byref(h)))
        return RefMatrix(self, h)

    def read_matrix_market(self, path):
        """the reference's read_matrix_market (inc/mm_io.hpp) -> (rp, ci, v)"""
        h = C.c_void_p()
        self.check(self.L.ref_read_mm(str(path).encode(), C.byref(h)))
        return RefMatrix(self, h).arrays()

    def write_matrix_market(self, A, path):
        m = self.matrix(A)  # keep the handle alive across the call
        self.check(self.L.ref_write_mm(m.h, str(path).encode()))

    def convdiff2d(self, nx, ny, bx, by, c):
        h = C.c_void_p()
        self.check(self.L.ref_convdiff2d(nx, ny, bx, by, c, C.byref(h)))
        return RefMatrix(self, h)

    # 3D generators (ref_capi.cpp: triplets through the reference's from_triplets)
    def stencil7(self, nx, ny, nz, diag, off):
        o = _d(off)
        h = C.c_void_p()
        self.check(self.L.ref_stencil7(nx, ny, nz, diag, o.ctypes.data_as(_D), C.byref(h)))
        return RefMatrix(self, h)

    def poisson3d(self, n):
        return self.stencil7(n, n, n, 6.0, [-1.0] * 6)

    def aniso3d(self, n, eps=1e-3):
        return self.stencil7(n, n, n, 4.0 + 2.0 * eps, [-1.0, -1.0, -1.0, -1.0, -eps, -eps])

    def convdiff3d(self, nx, ny, nz, bx, by, bz, c):
        h = C.c_void_p()
        self.check(self.L.ref_convdiff3d(nx, ny, nz, bx, by, bz, c, C.byref(h)))
        return RefMatrix(self, h)

    def stencil27(self, nx, ny, nz, diag=26.0, off=-1.0):
        h = C.c_void_p()
        self.check(self.L.ref_stencil27(nx, ny, nz, diag, off, C.byref(h)))
        return RefMatrix(self, h)

    def problem(self, name):
        """The BASELINE workloads, generated by the reference build."""
        if name == "C1":
            return self.convdiff2d(1024, 1024, 0.0, 0.0, 0.0)
        if name == "C2":
            return self.poisson3d(128)
        if name == "C3":
            return self.aniso3d(256, 1e-3)
        if name == "C4":
            return self.convdiff3d(256, 256, 256, 1.0, 100.0, 1.0, 1.0)
        if name == "T256":
            return self.poisson3d(256)
        if name == "P27_128":
            return self.stencil27(128, 128, 128)
        if name == "G128":
            return self.matrix(ArraysCsr(*graph_laplacian3d_arrays(128, seed=7)))
        raise ValueError(f"unknown problem {name}")

    def spmv(self, A, x):
        return self.matrix(A).spmv(x)

    def residual(self, A, x, f):
        return self.matrix(A).residual(x, f)

    def jacobi(self, A, omega, x, f, sweeps):
        return self.matrix(A).smooth(0, omega, x, f, sweeps)

    def node_hem(self, A):
        return self.matrix(A).node_hem()

    def hierarchy(self, A, coarse_target=500, max_levels=40):
        m = A if isinstance(A, RefMatrix) else self.matrix(A)
        return RefHier(self, m, coarse_target, max_levels)


class RefMatrix:
    def __init__(self, R: Ref, h):
        self.R, self.h = R, h

    def __del__(self):
        if getattr(self, "h", None):
            self.R.L.ref_csr_free(self.h)

    def arrays(self):
        n, m, z = C.c_int32(), C.c_int32(), C.c_int64()
        self.R.L.ref_csr_info(self.h, C.byref(n), C.byref(m), C.byref(z))
        rp = np.empty(n.value + 1, np.int32)
        ci = np.empty(z.value, np.int32)
        v = np.empty(z.value)
        self.R.L.ref_csr_copy(self.h, rp.ctypes.data_as(_I), ci.ctypes.data_as(_I), v.ctypes.data_as(_D))
        return rp, ci, v

    def nrows(self):
        return self._n()[0]

    def nnz(self):
        n, m, z = C.c_int32(), C.c_int32(), C.c_int64()
        self.R.L.ref_csr_info(self.h, C.byref(n), C.byref(m), C.byref(z))
        return z.value

    def _n(self):
        n, m, z = C.c_int32(), C.c_int32(), C.c_int64()
        self.R.L.ref_csr_info(self.h, C.byref(n), C.byref(m), C.byref(z))
        return n.value, m.value

    def spmv(self, x):
        x = _d(x)
        y = np.empty(self._n()[0])
        self.R.check(self.R.L.ref_spmv(self.h, x.ctypes.data_as(_D), y.ctypes.data_as(_D)))
        return y

    def residual(self, x, f):
        x, f = _d(x), _d(f)
        r = np.empty(self._n()[0])
        self.R.check(self.R.L.ref_residual(self.h, x.ctypes.data_as(_D), f.ctypes.data_as(_D),
                                           r.ctypes.data_as(_D)))
        return r

    def smooth(self, family, omega, x, f, sweeps):
        x = _d(x).copy()
        f = _d(f)
        self.R.check(self.R.L.ref_smooth(self.h, family, omega, x.ctypes.data_as(_D), f.ctypes.data_as(_D),
                                         sweeps))
        return x

    def node_hem(self):
        n = self._n()[0]
        out = np.empty(n, np.int32)
        nc = C.c_int32()
        self.R.check(self.R.L.ref_node_hem(self.h, out.ctypes.data_as(_I), C.byref(nc)))
        return out, nc.value


class RefHier:
    def __init__(self, R: Ref, m: RefMatrix, coarse_target, max_levels):
        self.R, self.m = R, m
        h = C.c_void_p()
        R.check(R.L.ref_hier_new(m.h, 0, coarse_target, max_levels, 0, C.byref(h)))
        self.h = h
        self.set_cycle()

    def __del__(self):
        if getattr(self, "h", None):
            self.R.L.ref_hier_free(self.h)
            self.h = None

    def nlevels(self):
        return self.R.L.ref_hier_nlevels(self.h)

    def level(self, k):
        n, nc = C.c_int32(), C.c_int32()
        z = C.c_int64()
        self.R.L.ref_hier_level_info(self.h, k, C.byref(n), C.byref(z), C.byref(nc))
        rp = np.empty(n.value + 1, np.int32)
        ci = np.empty(z.value, np.int32)
        v = np.empty(z.value)
        agg = np.empty(n.value, np.int32) if nc.value >= 0 else None
        self.R.L.ref_hier_level_copy(self.h, k, rp.ctypes.data_as(_I), ci.ctypes.data_as(_I),
                                     v.ctypes.data_as(_D), agg.ctypes.data_as(_I) if agg is not None else None)
        return rp, ci, v, agg

    def set_cycle(self, pre=6, post=6, omega=2.0 / 3.0, family=0):
        self.R.L.ref_hier_set_cycle(self.h, family, omega, pre, post)

    def memory_plan(self, scheme="MI"):
        """inc/memory_model.hpp plan_mi / plan_ci: (peak, resident after setup, per-cycle transfer) bytes."""
        pk, rs, pc = C.c_longlong(), C.c_longlong(), C.c_longlong()
        self.R.check(self.R.L.ref_memory_plan(self.h, 0 if scheme == "CI" else 1, C.byref(pk), C.byref(rs),
                                              C.byref(pc)))
        return pk.value, rs.value, pc.value

    def csr_bytes(self, k):
        """inc/memory_model.hpp csr_bytes of level k's matrix (8 B values, 4 B indices)."""
        return int(self.R.L.ref_csr_bytes(self.R.L.ref_hier_level_matrix(self.h, k)))

    def vcycle(self, f, x, k=0):
        f, x = _d(f), _d(x).copy()
        self.R.check(self.R.L.ref_vcycle(self.h, k, f.ctypes.data_as(_D), x.ctypes.data_as(_D)))
        return x

    def coarse_solve(self, f):
        f = _d(f)
        x = np.empty(f.size)
        self.R.check(self.R.L.ref_coarse_solve(self.h, f.ctypes.data_as(_D), x.ctypes.data_as(_D)))
        return x

    def _krylov(self, solver, b, tol, max_iters, amg):
        b = _d(b)
        x = np.empty(b.size)
        rep, hr, ht = _new_report(max(max_iters, 0) + 2)
        A0 = self.R.L.ref_hier_level_matrix(self.h, 0)
        self.R.check(self.R.L.ref_krylov(solver, A0, self.h if amg else None, b.ctypes.data_as(_D),
                                         x.ctypes.data_as(_D), tol, max_iters, C.byref(rep)))
        return SolveOut(x, rep, hr, ht)

    def pcg(self, b, tol, max_iters, amg=True):
        return self._krylov(0, b, tol, max_iters, amg)

    def pbicgstab(self, b, tol, max_iters, amg=True):
        return self._krylov(1, b, tol, max_iters, amg)

    def amg_solve(self, b, tol, max_cycles):
        b = _d(b)
        x = np.empty(b.size)
        rep, hr, ht = _new_report(max(max_cycles, 0) + 2)
        rc = self.R.L.ref_amg_solve(self.h, b.ctypes.data_as(_D), x.ctypes.data_as(_D), tol, max_cycles,
                                    C.byref(rep))
        out = SolveOut(x, rep, hr, ht)
        out.status = rc
        out.error = self.R.L.ref_last_error().decode() if rc else ""
        return out


def best_available():
    """The reference itself when its .so exists, else the restatement."""
    try:
        return Ref()
    except Exception:
        return Port()


def graph_laplacian3d_arrays(m, seed=7, shift=0.01):
    """(rp, ci, v) of bench.py's G128 operator (a 7-point graph Laplacian on m^3
    with random edge weights U[0.5, 1.5) + shift*I) in plain numpy, so the
    reference arm builds it without the product library. tests/test_oracle.py
    asserts it equals paper_2007_00056_b200.sparsh.graph_laplacian3d bit for bit."""
    n = m ** 3
    rng = np.random.default_rng(seed)
    idx = np.arange(n, dtype=np.int64).reshape(m, m, m)
    rows, cols, vals = [], [], []
    diag = np.full(n, shift)
    for ax in range(3):
        a = np.take(idx, np.arange(m - 1), axis=2 - ax).ravel()
        b = np.take(idx, np.arange(1, m), axis=2 - ax).ravel()
        w = rng.uniform(0.5, 1.5, a.size)
        rows += [a, b]
        cols += [b, a]
        vals += [-w, -w]
        np.add.at(diag, a, w)
        np.add.at(diag, b, w)
    r = np.concatenate(rows + [np.arange(n)])
    c = np.concatenate(cols + [np.arange(n)])
    v = np.concatenate(vals + [diag])
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp).astype(np.int32), c.astype(np.int32), v


class ArraysCsr:
    """Minimal CSR view (row_ptr/col_idx/values/nrows/ncols) for Ref.matrix()."""

    def __init__(self, rp, ci, v):
        self._rp, self._ci, self._v = rp, ci, v

    def row_ptr(self):
        return self._rp

    def col_idx(self):
        return self._ci

    def values(self):
        return self._v

    def nrows(self):
        return self._rp.size - 1

    def ncols(self):
        return self._rp.size - 1

    def nnz(self):
        return int(self._rp[-1])
