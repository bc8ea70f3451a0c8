"""Row partition of a hierarchy for multi-GPU solves (C ABI sb_partition*).

Every rank builds the same host hierarchy and calls ``Partition(h, rank,
nranks, gather_rows)``; the plans are identical on all ranks without any
communication. This module only exposes them; the device
solve consumes them inside libsparsh_b200.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check
from .sparsh import CycleParams, Hierarchy, SolveResult, _from_abi, _report


class Partition:
    def __init__(self, h: Hierarchy, rank: int, nranks: int, gather_rows: int):
        L = _lib.lib()
        p = C.c_void_p()
        check(L.sb_partition(h._h, int(rank), int(nranks), int(gather_rows), C.byref(p)))
        self._p = p
        self._h = h  # keep the hierarchy alive
        nl, fr = C.c_int(), C.c_int()
        check(L.sb_partition_info(p, C.byref(nl), C.byref(fr)))
        self.nlevels = nl.value
        self.first_replicated = fr.value
        self.rank, self.nranks = rank, nranks

    def __del__(self):
        try:
            if getattr(self, "_p", None):
                _lib.lib().sb_partition_free(self._p)
                self._p = None
        except Exception:
            pass

    def level(self, k: int) -> dict:
        info = (C.c_int64 * 11)()
        A = _lib.sb_csr()
        g, rg, xg = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
        m0, m1, par = C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)()
        check(_lib.lib().sb_partition_level(self._p, k, info, C.byref(A), C.byref(g), C.byref(rg), C.byref(xg),
                                            C.byref(m0), C.byref(m1), C.byref(par)))
        n_glob, lo, hi, ng, c_lo, c_hi, nrg, nxg, rep, wb, wa = list(info)

        def arr(ptr, n, dt):
            return np.ctypeslib.as_array(ptr, shape=(int(n),)).copy() if n else np.zeros(0, dt)

        nc_own = c_hi - c_lo
        # A's columns: window layout (wb > 0 or ghosts kept as c - lo) -> index x_ext[col + wb]
        # where x_ext = [wb rows below | own | wa rows above]; compact layout: wb = 0, [own | ghost]
        return dict(n_glob=n_glob, lo=lo, hi=hi, replicated=bool(rep), A=_from_abi(A), wb=wb, wa=wa,
                    ghost=arr(g, ng, np.int64), rghost=arr(rg, nrg, np.int64), xcghost=arr(xg, nxg, np.int64),
                    c_lo=c_lo, c_hi=c_hi,
                    mem0=arr(m0, nc_own if not rep else 0, np.int32), mem1=arr(m1, nc_own if not rep else 0, np.int32),
                    parent=arr(par, (hi - lo) if k + 1 < self.nlevels else 0, np.int32))

    def exchange(self, k: int, which: int) -> dict:
        """which: 0 x halo, 1 residual partners, 2 coarse parents."""
        cnt = (C.c_int64 * 4)()
        sp_, so, si = C.POINTER(C.c_int)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
        rp_, ro, rd = C.POINTER(C.c_int)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
        check(_lib.lib().sb_partition_exchange(self._p, k, which, cnt, C.byref(sp_), C.byref(so), C.byref(si),
                                               C.byref(rp_), C.byref(ro), C.byref(rd)))
        ns, nr, ts, tr = list(cnt)

        def arr(ptr, n, dt):
            return np.ctypeslib.as_array(ptr, shape=(int(n),)).copy() if n else np.zeros(0, dt)

        return dict(send_peers=arr(sp_, ns, np.int32), send_off=arr(so, ns + 1, np.int64),
                    send_idx=arr(si, ts, np.int32), recv_peers=arr(rp_, nr, np.int32),
                    recv_off=arr(ro, nr + 1, np.int64), recv_dst=arr(rd, nr, np.int64))


class DistSolver:
    """Partitioned device solve (C ABI sb_dist_*).

    local=True: `nranks` virtual ranks inside this process on one GPU (the
    exchanges are peer-buffer gathers) — b / x are GLOBAL vectors.
    local=False: this process is rank `rank` of `nranks` (one GPU each, NCCL);
    `nccl_id` is the 128-byte id from rank 0 (``nccl_unique_id()``); b / x are
    this rank's rows [lo, hi)."""

    def __init__(self, h: Hierarchy, nranks: int, gather_rows: int = 65536, *, local: bool = True,
                 rank: int = 0, nccl_id: bytes = None, device: int = 0, graphs: bool = True,
                 transport: str = "nccl"):
        """graphs (one rank per process): the whole solve captured as one CUDA graph
        with the exchanges inside (False: eager launches, host-evaluated conditions).
        transport: "nccl", or "p2p" (peer memory: gathers out of the peers' buffers,
        epoch flags; one rank per process needs p2p_export / p2p_connect)."""
        L = _lib.lib()
        d = C.c_void_p()
        opts = _lib.sb_device_opts(device, 1 if graphs else 0, -1, 0)
        self.transport = transport
        if local and transport == "p2p":
            check(L.sb_dist_create_local_p2p(h._h, int(nranks), int(gather_rows), C.byref(opts), C.byref(d)))
        elif local:
            check(L.sb_dist_create_local(h._h, int(nranks), int(gather_rows), C.byref(opts), C.byref(d)))
        elif transport == "p2p":
            check(L.sb_dist_create_p2p(h._h, int(rank), int(nranks), int(gather_rows), C.byref(opts), C.byref(d)))
        else:
            check(L.sb_dist_create(h._h, int(rank), int(nranks), nccl_id, int(gather_rows), C.byref(opts),
                                   C.byref(d)))
        self._d, self._h, self.local, self.nranks = d, h, local, nranks
        lo, hi, fr = C.c_int64(), C.c_int64(), C.c_int()
        check(L.sb_dist_rows(d, 0, C.byref(lo), C.byref(hi), C.byref(fr)))
        self.lo, self.hi, self.first_replicated = lo.value, hi.value, fr.value

    def __del__(self):
        try:
            if getattr(self, "_d", None):
                _lib.lib().sb_dist_destroy(self._d)
                self._d = None
        except Exception:
            pass

    def vcycle(self, f, p: CycleParams) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float64)
        x = np.zeros_like(f)
        cp = p._abi()
        check(_lib.lib().sb_dist_vcycle(self._d, C.byref(cp), _lib.dptr(f), _lib.dptr(x)))
        return x

    def _solve(self, fn, b, p, tol, max_iters, x_out=None):
        """b / x_out: numpy arrays (host) or integer device pointers (x_out required)."""
        cap = max(int(max_iters), 0) + 2
        hr, ht = np.zeros(cap), np.zeros(cap)
        rep = _lib.sb_report()
        rep.hist_cap = cap
        rep.residual_history = _lib.dptr(hr)
        rep.time_history = _lib.dptr(ht)
        cp = p._abi() if p is not None else None
        if isinstance(b, int):  # device pointers
            check(fn(self._d, C.byref(cp) if cp is not None else None, C.c_void_p(b), C.c_void_p(x_out),
                     float(tol), int(max_iters), C.byref(rep), 1))
            return SolveResult(None, _report(rep, hr, ht))
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b) if x_out is None else x_out
        check(fn(self._d, C.byref(cp) if cp is not None else None, b.ctypes.data_as(C.c_void_p),
                 x.ctypes.data_as(C.c_void_p), float(tol), int(max_iters), C.byref(rep), 0))
        return SolveResult(x, _report(rep, hr, ht))

    def pcg(self, b, p: CycleParams, tol, max_iters, x_out=None) -> SolveResult:
        return self._solve(_lib.lib().sb_dist_pcg, b, p, tol, max_iters, x_out)

    def pbicgstab(self, b, p: CycleParams, tol, max_iters, x_out=None) -> SolveResult:
        return self._solve(_lib.lib().sb_dist_pbicgstab, b, p, tol, max_iters, x_out)

    def p2p_export(self) -> bytes:
        """This rank's IPC handle blob (every rank needs every rank's, in rank order)."""
        L = _lib.lib()
        n = C.c_int64()
        check(L.sb_dist_p2p_export(self._d, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(L.sb_dist_p2p_export(self._d, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def p2p_connect(self, blobs) -> None:
        """blobs: every rank's p2p_export() in rank order (equal lengths)."""
        each = len(blobs[0])
        if any(len(b) != each for b in blobs):
            raise ValueError("p2p_connect: blobs of different lengths")
        check(_lib.lib().sb_dist_p2p_connect(self._d, b"".join(blobs), each))

    def last_solve_ms(self) -> float:
        return float(_lib.lib().sb_dist_last_solve_ms(self._d))

    def last_launches(self) -> int:
        return int(_lib.lib().sb_dist_last_launches(self._d))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(_lib.lib().sb_nccl_unique_id(buf))
    return buf.raw
