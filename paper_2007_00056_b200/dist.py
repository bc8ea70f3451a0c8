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
from .sparsh import Hierarchy, _from_abi


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
        info = (C.c_int64 * 9)()
        A = _lib.sb_csr()
        g, rg, xg = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
        m0, m1, par = C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)()
        check(_lib.lib().sb_partition_level(self._p, k, info, C.byref(A), C.byref(g), C.byref(rg), C.byref(xg),
                                            C.byref(m0), C.byref(m1), C.byref(par)))
        n_glob, lo, hi, ng, c_lo, c_hi, nrg, nxg, rep = list(info)

        def arr(ptr, n, dt):
            return np.ctypeslib.as_array(ptr, shape=(int(n),)).copy() if n else np.zeros(0, dt)

        nc_own = c_hi - c_lo
        return dict(n_glob=n_glob, lo=lo, hi=hi, replicated=bool(rep), A=_from_abi(A),
                    ghost=arr(g, ng, np.int64), rghost=arr(rg, nrg, np.int64), xcghost=arr(xg, nxg, np.int64),
                    c_lo=c_lo, c_hi=c_hi,
                    mem0=arr(m0, nc_own if not rep else 0, np.int32), mem1=arr(m1, nc_own if not rep else 0, np.int32),
                    parent=arr(par, (hi - lo) if k + 1 < self.nlevels else 0, np.int32))

    def exchange(self, k: int, which: int) -> dict:
        """which: 0 x halo, 1 residual partners, 2 coarse parents."""
        cnt = (C.c_int64 * 4)()
        sp_, so, si = C.POINTER(C.c_int)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
        rp_, ro = C.POINTER(C.c_int)(), C.POINTER(C.c_int64)()
        check(_lib.lib().sb_partition_exchange(self._p, k, which, cnt, C.byref(sp_), C.byref(so), C.byref(si),
                                               C.byref(rp_), C.byref(ro)))
        ns, nr, ts, tr = list(cnt)

        def arr(ptr, n, dt):
            return np.ctypeslib.as_array(ptr, shape=(int(n),)).copy() if n else np.zeros(0, dt)

        return dict(send_peers=arr(sp_, ns, np.int32), send_off=arr(so, ns + 1, np.int64),
                    send_idx=arr(si, ts, np.int32), recv_peers=arr(rp_, nr, np.int32),
                    recv_off=arr(ro, nr + 1, np.int64))
