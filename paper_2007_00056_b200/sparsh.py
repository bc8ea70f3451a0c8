"""Python mirror of the reference's solve-phase API (sparsh, inc/*.hpp), backed
by the B200 C ABI (include/sparsh_b200.h). Names, argument meaning and error
behaviour follow the reference so tests read like its own:

    A = poisson2d(64, 64)
    cfg = SolverConfig(smoother=SmootherKind.weighted_jacobi(), max_levels=40)
    h = Hierarchy(A, cfg)                                  # hierarchy.hpp:51
    res = pcg(A, rhs_ones(A.nrows()),
              make_amg_preconditioner(h, CycleParams.from_config(cfg)),
              1e-8, 1000)                                  # krylov.hpp:65

Setup (node-HEM + Galerkin + coarse LU) runs on the host in C++ and is
bit-exact with the reference; everything on the solve path runs on the GPU.
std::invalid_argument maps to InvalidArgument (a ValueError), runtime_error to
RuntimeError. There is no CPU fallback: GPU entry points raise if the CUDA
library or device is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import InvalidArgument, CudaError, check, dptr, iptr, lptr

__all__ = [
    "CsrMatrix", "Aggregation", "Level", "Hierarchy", "HierarchyStats", "SolverConfig",
    "SmootherKind", "CycleParams", "Preconditioner", "Termination", "ConvergenceReport",
    "SolveResult", "InvalidArgument", "CudaError", "make_amg_preconditioner", "vcycle",
    "vcycle_in_place", "amg_solve", "pcg", "pbicgstab", "cg", "bicgstab", "spmv",
    "residual", "smooth", "smooth_in_place", "stats", "convdiff2d", "poisson2d",
    "poisson3d", "aniso3d", "convdiff3d", "poisson3d_27", "graph_laplacian3d", "rhs_ones", "rhs_random", "zeros",
]


# --------------------------------------------------------------------------
# CSR matrix (inc/csr.hpp:44-169)
# --------------------------------------------------------------------------
class CsrMatrix:
    """Immutable CSR matrix: int32 columns strictly increasing per row, f64 values."""

    def __init__(self, nrows, ncols, row_ptr, col_idx, values, _validate=True):
        self._n = int(nrows)
        self._m = int(ncols)
        rp = np.ascontiguousarray(row_ptr)
        self._rp = rp.astype(np.int64 if rp.size and rp[-1] > np.iinfo(np.int32).max else np.int32, copy=False)
        self._ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        self._v = np.ascontiguousarray(values, dtype=np.float64)
        self._plain = None
        if _validate:
            self._validate()

    def _validate(self):  # csr.hpp:135-162
        if self._n < 0 or self._m < 0:
            raise InvalidArgument("CsrMatrix: negative dimension")
        if self._rp.size != self._n + 1:
            raise InvalidArgument("CsrMatrix: row_ptr length mismatch")
        if self._rp[0] != 0:
            raise InvalidArgument("CsrMatrix: row_ptr[0] != 0")
        if self._rp[-1] != self._ci.size:
            raise InvalidArgument("CsrMatrix: row_ptr[nrows] != nnz")
        if self._ci.size != self._v.size:
            raise InvalidArgument("CsrMatrix: col/value length mismatch")
        d = np.diff(self._rp.astype(np.int64))
        if (d < 0).any():
            raise InvalidArgument("CsrMatrix: row_ptr not monotone")
        if self._ci.size:
            bad = (self._ci < 0) | (self._ci >= self._m)
            if bad.any():
                row = int(np.searchsorted(self._rp, np.argmax(bad), side="right") - 1)
                raise InvalidArgument(f"CsrMatrix: column index out of range in row {row}")
            rows = np.repeat(np.arange(self._n), d)
            inc = np.diff(self._ci.astype(np.int64)) <= 0
            same = rows[1:] == rows[:-1]
            if (inc & same).any():
                row = int(rows[1:][inc & same][0])
                raise InvalidArgument(f"CsrMatrix: columns not strictly increasing in row {row}")

    @staticmethod
    def from_triplets(nrows, ncols, entries):
        """csr.hpp:57-95: sort by (row, col), sum duplicates (0.0 + v + ...)."""
        ent = list(entries)
        for (r, c, _) in ent:
            if r < 0 or r >= nrows or c < 0 or c >= ncols:
                raise InvalidArgument(f"from_triplets: entry ({r}, {c}) outside {nrows}x{ncols}")
        ent.sort(key=lambda t: (t[0], t[1]))
        rp = np.zeros(nrows + 1, dtype=np.int64)
        cols, vals = [], []
        k = 0
        while k < len(ent):
            r, c = ent[k][0], ent[k][1]
            s = 0.0
            while k < len(ent) and ent[k][0] == r and ent[k][1] == c:
                s += float(ent[k][2])
                k += 1
            cols.append(c)
            vals.append(s)
            rp[r + 1] = len(cols)
        for r in range(nrows):
            rp[r + 1] = max(rp[r + 1], rp[r])
        return CsrMatrix(nrows, ncols, rp, np.array(cols, dtype=np.int32), np.array(vals, dtype=np.float64))

    @staticmethod
    def from_dense(a):
        a = np.asarray(a, dtype=np.float64)
        n, m = a.shape
        ent = [(i, j, a[i, j]) for i in range(n) for j in range(m) if a[i, j] != 0.0]
        return CsrMatrix.from_triplets(n, m, ent)

    @staticmethod
    def identity(n):
        return CsrMatrix(n, n, np.arange(n + 1), np.arange(n, dtype=np.int32), np.ones(n))

    def nrows(self):
        return self._n

    def ncols(self):
        return self._m

    def nnz(self):
        return int(self._ci.size)

    def is_square(self):
        return self._n == self._m

    def row_ptr(self):
        return self._rp

    def col_idx(self):
        return self._ci

    def values(self):
        return self._v

    def to_dense(self):
        a = np.zeros((self._n, self._m))
        rows = np.repeat(np.arange(self._n), np.diff(self._rp.astype(np.int64)))
        a[rows, self._ci] = self._v
        return a

    def __eq__(self, o):
        return (isinstance(o, CsrMatrix) and self._n == o._n and self._m == o._m
                and np.array_equal(self._rp.astype(np.int64), o._rp.astype(np.int64))
                and np.array_equal(self._ci, o._ci) and np.array_equal(self._v, o._v))

    def _abi(self) -> _lib.sb_csr:
        s = _lib.sb_csr()
        s.nrows, s.ncols = self._n, self._m
        if self._rp.dtype == np.int32:
            s.row_ptr32 = iptr(self._rp)
        else:
            s.row_ptr64 = lptr(self._rp)
        s.col_idx = iptr(self._ci)
        s.values = dptr(self._v)
        return s

    def _device(self) -> "Hierarchy":
        """Single-level device context for matrix-only calls (spmv, cg, ...)."""
        if self._plain is None:
            self._plain = Hierarchy(self, SolverConfig(max_levels=1, coarse_target=1), _coarse_solver=-1)
        return self._plain


def _from_abi(s: _lib.sb_csr) -> CsrMatrix:
    n = int(s.nrows)
    if s.row_ptr32:
        rp = np.ctypeslib.as_array(s.row_ptr32, shape=(n + 1,)).copy()
    else:
        rp = np.ctypeslib.as_array(s.row_ptr64, shape=(n + 1,)).copy()
    nnz = int(rp[-1])
    ci = np.ctypeslib.as_array(s.col_idx, shape=(nnz,)).copy() if nnz else np.zeros(0, np.int32)
    v = np.ctypeslib.as_array(s.values, shape=(nnz,)).copy() if nnz else np.zeros(0)
    return CsrMatrix(n, int(s.ncols), rp, ci, v, _validate=False)


# --------------------------------------------------------------------------
# config (inc/smoother.hpp:22-49, inc/config.hpp:81-105, inc/cycle.hpp:24-32)
# --------------------------------------------------------------------------
default_jacobi_omega = 2.0 / 3.0


@dataclass(frozen=True)
class SmootherKind:
    family: str = "gauss_seidel_symmetric"
    omega: float = default_jacobi_omega

    @staticmethod
    def weighted_jacobi(omega: float = default_jacobi_omega) -> "SmootherKind":
        if not (omega > 0.0) or omega > 1.0:
            raise InvalidArgument(f"SmootherKind: Jacobi weight {omega:f} outside (0, 1]")
        return SmootherKind("weighted_jacobi", float(omega))

    @staticmethod
    def gauss_seidel_forward():
        return SmootherKind("gauss_seidel_forward")

    @staticmethod
    def gauss_seidel_backward():
        return SmootherKind("gauss_seidel_backward")

    @staticmethod
    def gauss_seidel_symmetric():
        return SmootherKind("gauss_seidel_symmetric")

    def _code(self):
        return {"weighted_jacobi": 0, "gauss_seidel_forward": 1,
                "gauss_seidel_backward": 2, "gauss_seidel_symmetric": 3}[self.family]


@dataclass
class SolverConfig:
    coarsening: str = "node_hem"
    smoother: SmootherKind = field(default_factory=SmootherKind.gauss_seidel_symmetric)
    pre_sweeps: int = 6
    post_sweeps: int = 6
    coarse_target: int = 500
    max_levels: int = 10
    tol: float = 1e-8
    max_iters: int = 1000
    solver: str = "amg"
    coarse_solver: str = "direct"

    def validate(self):  # config.hpp:93-104
        if not (self.tol > 0.0):
            raise InvalidArgument("SolverConfig: tol must be > 0")
        if self.pre_sweeps < 0 or self.post_sweeps < 0:
            raise InvalidArgument("SolverConfig: sweep counts must be >= 0")
        if self.coarse_target < 1:
            raise InvalidArgument("SolverConfig: coarse_target must be >= 1")
        if self.max_levels < 1:
            raise InvalidArgument("SolverConfig: max_levels must be >= 1")
        if self.max_iters < 0:
            raise InvalidArgument("SolverConfig: max_iters must be >= 0")


@dataclass
class CycleParams:
    pre_sweeps: int = 6
    post_sweeps: int = 6
    smoother: SmootherKind = field(default_factory=SmootherKind.gauss_seidel_symmetric)

    @staticmethod
    def from_config(cfg: SolverConfig) -> "CycleParams":
        return CycleParams(cfg.pre_sweeps, cfg.post_sweeps, cfg.smoother)

    def _abi(self) -> _lib.sb_cycle:
        return _lib.sb_cycle(self.pre_sweeps, self.post_sweeps, self.smoother._code(), self.smoother.omega)


class Termination(enum.IntEnum):  # convergence.hpp:15
    converged = 0
    max_iters = 1
    breakdown = 2
    diverged = 3


@dataclass
class ConvergenceReport:  # convergence.hpp:33-42
    residual_history: List[float] = field(default_factory=list)
    time_history: List[float] = field(default_factory=list)
    iterations: int = 0
    termination: Termination = Termination.max_iters
    wall_time: float = 0.0
    true_residual: float = 0.0

    def converged(self):
        return self.termination == Termination.converged


@dataclass
class SolveResult:
    x: np.ndarray
    report: ConvergenceReport


@dataclass
class Aggregation:  # aggregation.hpp:24-61
    fine_to_coarse: np.ndarray
    n_coarse: int

    def n_fine(self):
        return int(self.fine_to_coarse.size)


@dataclass
class Level:  # hierarchy.hpp:24-28
    A: CsrMatrix
    agg: Optional[Aggregation]

    @property
    def P_to_coarser(self) -> Optional[CsrMatrix]:
        """prolongation_from_aggregation (aggregation.hpp:68-82)."""
        if self.agg is None:
            return None
        n = self.agg.n_fine()
        return CsrMatrix(n, self.agg.n_coarse, np.arange(n + 1), self.agg.fine_to_coarse, np.ones(n))


@dataclass
class HierarchyStats:
    levels: list
    operator_complexity: float
    grid_complexity: float
    coarsening_stalled: bool


# --------------------------------------------------------------------------
# Hierarchy (inc/hierarchy.hpp:49-93) — host setup + lazily created device context
# --------------------------------------------------------------------------
class Hierarchy:
    def __init__(self, A: CsrMatrix, cfg: SolverConfig = None, device: int = 0, *, _coarse_solver=None,
                 coarse_exact: bool = False, galerkin_gpu: bool = False, host_levels_from: int = -1,
                 graphs: bool = True):
        cfg = cfg or SolverConfig()
        if not A.is_square():
            raise InvalidArgument("Hierarchy: matrix must be square")
        cfg.validate()
        if cfg.coarsening != "node_hem":
            raise InvalidArgument("Hierarchy: only node_hem coarsening is provided on the device path")
        if cfg.coarse_solver != "direct" and _coarse_solver is None:
            raise InvalidArgument("Hierarchy: coarse_solver=cg is not supported on the device path")
        L = _lib.lib()
        opts = _lib.sb_setup_opts(0, cfg.coarse_target, cfg.max_levels,
                                  0 if _coarse_solver is None else _coarse_solver, 0,
                                  1 if galerkin_gpu else 0, device)
        h = C.c_void_p()
        a = A._abi()
        check(L.sb_setup(C.byref(a), C.byref(opts), C.byref(h)))
        self._h = h
        self._ctx = None
        self._device = device
        self._coarse_exact = bool(coarse_exact)
        self._host_from = int(host_levels_from)  # hybrid mode
        self._graphs = bool(graphs)  # False: eager launches, host-side loop control (sb_device_opts.use_graphs)
        self._levels = None
        self._A0 = A
        self.config = cfg

    @classmethod
    def from_stencil27(cls, nx: int, ny: int, nz: int, diag: float, off: float, cfg: SolverConfig = None,
                       device: int = 0, galerkin_gpu: bool = False, host_levels_from: int = -1) -> "Hierarchy":
        """Hierarchy of the 3D 27-point operator generated straight into the setup's
        host storage (sb_setup_stencil27): no Python-side copy of the fine matrix,
        int64 row offsets (config 5: 512^3, nnz 3.6e9). host_levels_from: hybrid
        placement of the coarse levels (as in __init__)."""
        cfg = cfg or SolverConfig()
        cfg.validate()
        self = cls.__new__(cls)
        opts = _lib.sb_setup_opts(0, cfg.coarse_target, cfg.max_levels, 0, 0, 1 if galerkin_gpu else 0, device)
        h = C.c_void_p()
        check(_lib.lib().sb_setup_stencil27(int(nx), int(ny), int(nz), float(diag), float(off), C.byref(opts),
                                            C.byref(h)))
        self._h, self._ctx, self._device, self._coarse_exact, self._graphs = h, None, device, False, True
        self._host_from, self._levels, self._A0, self.config = int(host_levels_from), None, None, cfg
        return self

    def __del__(self):
        try:
            L = _lib.lib()
            if getattr(self, "_ctx", None):
                L.sb_destroy(self._ctx)
                self._ctx = None
            if getattr(self, "_h", None):
                L.sb_hier_free(self._h)
                self._h = None
        except Exception:
            pass

    def nlevels(self) -> int:
        return _lib.lib().sb_hier_nlevels(self._h)

    def coarsening_stalled(self) -> bool:
        return bool(_lib.lib().sb_hier_stalled(self._h))

    def levels(self) -> List[Level]:
        if self._levels is None:
            out = []
            for k in range(self.nlevels()):
                s = _lib.sb_csr()
                agg_p = C.POINTER(C.c_int32)()
                nc = C.c_int64()
                check(_lib.lib().sb_hier_level(self._h, k, C.byref(s), C.byref(agg_p), C.byref(nc)))
                A = _from_abi(s)
                agg = None
                if agg_p:
                    agg = Aggregation(np.ctypeslib.as_array(agg_p, shape=(A.nrows(),)).copy(), int(nc.value))
                out.append(Level(A, agg))
            self._levels = out
        return self._levels

    def level(self, k: int) -> Level:
        if k < 0 or k >= self.nlevels():
            raise IndexError("level out of range")
        return self.levels()[k]

    def coarsest(self) -> CsrMatrix:
        return self.level(self.nlevels() - 1).A

    def coarse_counts(self):
        s, n, c = C.c_long(), C.c_long(), C.c_long()
        check(_lib.lib().sb_hier_coarse_counts(self._h, C.byref(s), C.byref(n), C.byref(c)))
        return s.value, n.value, c.value

    # -- device side -------------------------------------------------------
    def ctx(self):
        if self._ctx is None:
            c = C.c_void_p()
            opts = _lib.sb_device_opts(self._device, 1 if self._graphs else 0, self._host_from,
                                       int(self._coarse_exact))
            check(_lib.lib().sb_create(self._h, C.byref(opts), C.byref(c)))
            self._ctx = c
        return self._ctx

    def last_solve_launches(self) -> int:
        """Kernels the last solve executed (sb_last_solve_launches)."""
        return int(_lib.lib().sb_last_solve_launches(self.ctx()))

    def device_bytes(self) -> int:
        return int(_lib.lib().sb_device_bytes(self.ctx()))

    def host_bytes(self) -> int:
        """Hybrid mode: level storage held in pinned host memory."""
        return int(_lib.lib().sb_host_bytes(self.ctx()))

    def _n(self, k):
        return self.level(k).A.nrows()

    def spmv(self, k, x):
        x = _vec(x, self.level(k).A.ncols(), "spmv")
        y = np.empty(self._n(k))
        check(_lib.lib().sb_spmv(self.ctx(), k, dptr(x), dptr(y)))
        return y

    def residual(self, k, x, f):
        n = self._n(k)
        x, f = _vec(x, n, "residual"), _vec(f, n, "residual")
        r = np.empty(n)
        check(_lib.lib().sb_residual(self.ctx(), k, dptr(x), dptr(f), dptr(r)))
        return r

    def smooth(self, k, kind: SmootherKind, x, f, sweeps):
        n = self._n(k)
        x = _vec(x, n, "smooth").copy()
        f = _vec(f, n, "smooth")
        cp = _lib.sb_cycle(0, 0, kind._code(), kind.omega)
        check(_lib.lib().sb_smooth(self.ctx(), k, C.byref(cp), dptr(x), dptr(f), int(sweeps)))
        return x

    def restrict(self, k, r):
        lv = self.level(k)
        if lv.agg is None:
            raise InvalidArgument("restrict: coarsest level has no aggregation")
        r = _vec(r, lv.A.nrows(), "restrict")
        fc = np.empty(lv.agg.n_coarse)
        check(_lib.lib().sb_restrict(self.ctx(), k, dptr(r), dptr(fc)))
        return fc

    def prolong_add(self, k, xc, x):
        lv = self.level(k)
        xc = _vec(xc, lv.agg.n_coarse, "prolong")
        x = _vec(x, lv.A.nrows(), "prolong").copy()
        check(_lib.lib().sb_prolong(self.ctx(), k, dptr(xc), dptr(x)))
        return x

    def coarse_solve(self, f):
        n = self.coarsest().nrows()
        f = _vec(f, n, "CoarseFactorization::solve")
        x = np.empty(n)
        check(_lib.lib().sb_coarse_solve(self.ctx(), dptr(f), dptr(x)))
        return x


def read_matrix_market(path) -> CsrMatrix:
    """mm_io.hpp:35-111 (reference semantics and messages)."""
    return _gen(_lib.lib().sb_read_matrix_market, str(path).encode())


def write_matrix_market(A: CsrMatrix, path) -> None:
    """mm_io.hpp:114-135."""
    a = A._abi()
    check(_lib.lib().sb_write_matrix_market(str(path).encode(), C.byref(a)))


def galerkin_product_gpu(A: CsrMatrix, agg: "Aggregation", device: int = 0) -> CsrMatrix:
    """galerkin_product(A, agg) (inc/aggregation.hpp:92-152) computed on the GPU;
    bit-identical to the reference."""
    f2c = np.ascontiguousarray(agg.fine_to_coarse, dtype=np.int32)
    out = _lib.sb_csr()
    a = A._abi()
    L = _lib.lib()
    check(L.sb_galerkin_gpu(C.byref(a), f2c.ctypes.data_as(C.POINTER(C.c_int32)), int(agg.n_coarse), int(device),
                            C.byref(out)))
    try:
        return _from_abi(out)
    finally:
        L.sb_free_csr(C.byref(out))


def stats(h: Hierarchy) -> HierarchyStats:  # hierarchy.hpp:99-113
    lv = [(l.A.nrows(), l.A.nnz()) for l in h.levels()]
    nnz0, n0 = float(lv[0][1]), float(lv[0][0])
    return HierarchyStats(lv, sum(z for _, z in lv) / nnz0 if nnz0 > 0 else 1.0,
                          sum(n for n, _ in lv) / n0 if n0 > 0 else 1.0, h.coarsening_stalled())


def _vec(x, n, who):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 1 or x.size != n:
        raise InvalidArgument(f"{who}: vector length {x.size} does not match dimension {n}")
    return x


# --------------------------------------------------------------------------
# solve phase (inc/cycle.hpp, inc/krylov.hpp)
# --------------------------------------------------------------------------
@dataclass
class Preconditioner:  # krylov.hpp:30-36; AMG = cycle.hpp:137-145
    kind: str
    hierarchy: Optional[Hierarchy] = None
    params: Optional[CycleParams] = None

    @staticmethod
    def identity() -> "Preconditioner":
        return Preconditioner("identity")

    def apply(self, r):
        if self.kind == "identity":
            return np.array(r, dtype=np.float64, copy=True)
        return vcycle(self.hierarchy, 0, r, zeros(len(r)), self.params)


def make_amg_preconditioner(h: Hierarchy, p: CycleParams = None) -> Preconditioner:
    return Preconditioner("amg", h, p if p is not None else CycleParams())


def vcycle_in_place(h: Hierarchy, k: int, f, x: np.ndarray, p: CycleParams = None):
    """cycle.hpp:53-75 (x updated in place)."""
    p = p if p is not None else CycleParams()
    n = h.level(k).A.nrows()
    f = np.ascontiguousarray(f, dtype=np.float64)
    if f.size != n or x.size != n:
        raise InvalidArgument(f"vcycle: vector lengths ({f.size}, {x.size}) do not match level size {n}")
    xx = np.ascontiguousarray(x, dtype=np.float64).copy()
    cp = p._abi()
    check(_lib.lib().sb_vcycle(h.ctx(), C.byref(cp), k, dptr(f), dptr(xx)))
    x[...] = xx


def vcycle(h: Hierarchy, k: int, f, x, p: CycleParams = None) -> np.ndarray:
    x = np.array(x, dtype=np.float64, copy=True)
    vcycle_in_place(h, k, f, x, p)
    return x


def _report(rep: _lib.sb_report, hist_r, hist_t) -> ConvergenceReport:
    m = min(rep.hist_len, rep.hist_cap)
    return ConvergenceReport(list(hist_r[:m]), list(hist_t[:m]), rep.iterations,
                             Termination(rep.termination), rep.wall_time, rep.true_residual)


def _solve(fn, ctx, cp, b, tol, max_iters):
    n = b.size
    x = np.empty(n)
    cap = max(int(max_iters), 0) + 2
    hr, ht = np.zeros(cap), np.zeros(cap)
    rep = _lib.sb_report()
    rep.hist_cap = cap
    rep.residual_history = dptr(hr)
    rep.time_history = dptr(ht)
    rc = fn(ctx, C.byref(cp) if cp is not None else None, dptr(b), dptr(x), float(tol), int(max_iters),
            C.byref(rep))
    return rc, x, _report(rep, hr, ht)


def _krylov(which, A: CsrMatrix, b, M: Preconditioner, tol, max_iters) -> SolveResult:
    if not A.is_square():
        raise InvalidArgument(f"{which}: matrix must be square")
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != A.nrows():
        raise InvalidArgument(f"{which}: rhs length {b.size} does not match dimension {A.nrows()}")
    if not (tol > 0.0):
        raise InvalidArgument(f"{which}: tol must be > 0")
    if M.kind == "identity":
        h, cp = A._device(), None
    else:
        h, cp = M.hierarchy, M.params._abi()
        if h.level(0).A is not A and not (h.level(0).A == A):
            raise InvalidArgument(f"{which}: the AMG preconditioner was built for a different matrix")
    L = _lib.lib()
    fn = L.sb_pcg if which == "pcg" else L.sb_pbicgstab
    rc, x, rep = _solve(fn, h.ctx(), cp, b, tol, max_iters)
    check(rc)
    return SolveResult(x, rep)


def pcg(A, b, M, tol, max_iters) -> SolveResult:
    return _krylov("pcg", A, b, M, tol, max_iters)


def pbicgstab(A, b, M, tol, max_iters) -> SolveResult:
    return _krylov("pbicgstab", A, b, M, tol, max_iters)


def cg(A, b, tol, max_iters) -> SolveResult:
    return pcg(A, b, Preconditioner.identity(), tol, max_iters)


def bicgstab(A, b, tol, max_iters) -> SolveResult:
    return pbicgstab(A, b, Preconditioner.identity(), tol, max_iters)


def amg_solve(h: Hierarchy, b, tol, max_cycles, p: CycleParams = None) -> SolveResult:
    """cycle.hpp:91-130; raises RuntimeError('amg_solve: diverged ...')."""
    p = p if p is not None else CycleParams()
    n = h.level(0).A.nrows()
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != n:
        raise InvalidArgument(f"amg_solve: rhs length {b.size} does not match dimension {n}")
    if not (tol > 0.0):
        raise InvalidArgument("amg_solve: tol must be > 0")
    rc, x, rep = _solve(_lib.lib().sb_amg_solve, h.ctx(), p._abi(), b, tol, max_cycles)
    check(rc)
    return SolveResult(x, rep)


# matrix-only kernels (csr.hpp / smoother.hpp) on a single-level device context
def spmv(A: CsrMatrix, x) -> np.ndarray:
    return A._device().spmv(0, x)


def residual(A: CsrMatrix, x, f) -> np.ndarray:
    return A._device().residual(0, x, f)


def smooth(kind: SmootherKind, A: CsrMatrix, x, f, sweeps) -> np.ndarray:
    if not A.is_square():
        raise InvalidArgument("smooth: matrix must be square")
    return A._device().smooth(0, kind, x, f, sweeps)


def smooth_in_place(kind, A, x, f, sweeps):
    x[...] = smooth(kind, A, x, f, sweeps)


# --------------------------------------------------------------------------
# problems (inc/problems.hpp + the 3D harness generators of SURVEY.md §8d)
# --------------------------------------------------------------------------
def _gen(fn, *args) -> CsrMatrix:
    s = _lib.sb_csr()
    check(fn(*args, C.byref(s)))
    try:
        return _from_abi(s)
    finally:
        _lib.lib().sb_free_csr(C.byref(s))


def convdiff2d(nx, ny, bx, by, c) -> CsrMatrix:
    return _gen(_lib.lib().sb_gen_convdiff2d, nx, ny, bx, by, c)


def poisson2d(nx, ny) -> CsrMatrix:
    return convdiff2d(nx, ny, 0.0, 0.0, 0.0)


def stencil7(nx, ny, nz, diag, off) -> CsrMatrix:
    o = np.ascontiguousarray(off, dtype=np.float64)
    return _gen(_lib.lib().sb_gen_stencil7, nx, ny, nz, float(diag), dptr(o))


def poisson3d(n, ny=None, nz=None) -> CsrMatrix:
    """7-point Poisson, integer stencil (6, -1) = cell-volume scaling x 1/h."""
    return stencil7(n, ny or n, nz or n, 6.0, [-1.0] * 6)


def aniso3d(n, eps=1e-3) -> CsrMatrix:
    """7-point anisotropic diffusion, eps in z: (4 + 2 eps, -1 in x/y, -eps in z)."""
    return stencil7(n, n, n, 4.0 + 2.0 * eps, [-1.0, -1.0, -1.0, -1.0, -eps, -eps])


def convdiff3d(nx, ny, nz, bx, by, bz, c) -> CsrMatrix:
    return _gen(_lib.lib().sb_gen_convdiff3d, nx, ny, nz, bx, by, bz, c)


def graph_laplacian3d(m, seed=7, shift=0.01) -> CsrMatrix:
    """SPD graph Laplacian of the m^3 7-point grid with random edge weights
    U[0.5, 1.5) plus shift*I: no two rows share their values, so no level has
    row patterns and the hierarchy is irregular (node-HEM on random weights)."""
    n = m ** 3
    rng = np.random.default_rng(seed)
    idx = np.arange(n, dtype=np.int64).reshape(m, m, m)  # [z, y, x]
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
    return CsrMatrix(n, n, np.cumsum(rp), c.astype(np.int32), v)


def poisson3d_27(n) -> CsrMatrix:
    return _gen(_lib.lib().sb_gen_stencil27, n, n, n, 26.0, -1.0)


def rhs_ones(n) -> np.ndarray:
    return np.ones(int(n))


def rhs_random(n, seed=42) -> np.ndarray:
    out = np.empty(int(n))
    check(_lib.lib().sb_gen_rhs_random(int(n), int(seed), dptr(out)))
    return out


def zeros(n) -> np.ndarray:
    return np.zeros(int(n))
