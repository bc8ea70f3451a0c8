"""keep the reference's setup, accelerate only the solve.

oracle/_ref/adopt_reference (tests/cpp/adopt_reference.cpp, compiled against
the reference headers and libsparsh_b200.so) builds sparsh::Hierarchy with the
reference (inc/hierarchy.hpp:51), hands its levels to sb_hier_from_levels and
solves with sb_pcg; it also runs the reference's own pcg and the product's own
setup on the same matrix."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

EXE = os.path.join(ROOT, "oracle", "_ref", "adopt_reference")


@pytest.mark.gpu
def test_reference_hierarchy_adopted():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/adopt_reference not built (needs the reference headers at build time)")
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["adopted_converged"] == 1
    assert d["adopted_eq_setup_bitwise"] == 1          # adopted == sb_setup, bit for bit
    assert abs(d["adopted_iters"] - d["ref_iters"]) <= 1
    assert d["rel_err_equal_iters"] < 1e-10
    assert d["bad_agg_rejected"] == 1


def test_hier_from_levels_validates_aggregation(sp):
    """Aggregation::validate (inc/aggregation.hpp:42-58) on adoption: a coarse node
    with 3 or 0 fine nodes is rejected with the reference's message (host only)."""
    import ctypes as C
    import numpy as np
    from paper_2007_00056_b200 import _lib

    A = sp.poisson2d(8, 8)
    agg, nc = np.arange(64, dtype=np.int32) // 2, 32
    Ac = sp.CsrMatrix.identity(nc)

    def adopt(f2c):
        ls = (_lib.sb_csr * 2)(A._abi(), Ac._abi())
        arr = np.ascontiguousarray(f2c, dtype=np.int32)
        ptrs = (C.POINTER(C.c_int32) * 1)(arr.ctypes.data_as(C.POINTER(C.c_int32)))
        h = C.c_void_p()
        rc = _lib.lib().sb_hier_from_levels(2, ls, ptrs, C.byref(h))
        if rc == 0:
            _lib.lib().sb_hier_free(h)
        return rc, _lib.lib().sb_last_error().decode()

    assert adopt(agg)[0] == 0
    bad = agg.copy()
    bad[2] = 0  # coarse node 0 gets 3 fine nodes, node 1 keeps one
    rc, msg = adopt(bad)
    assert rc == 1 and msg == "Aggregation: coarse node 0 has 3 fine nodes"
    bad = agg.copy()
    bad[2:4] = 0
    bad[0:2] = 1  # coarse node 0: {2, 3}, node 1: {0, 1} ... then make node 5 empty
    bad[10:12] = 4
    rc, msg = adopt(bad)
    assert rc == 1 and msg == "Aggregation: coarse node 4 has 4 fine nodes"
    bad = agg.copy()
    bad[5] = 40
    rc, msg = adopt(bad)
    assert rc == 1 and msg == "Aggregation: coarse index 40 outside [0, 32)"
