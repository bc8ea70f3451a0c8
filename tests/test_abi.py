"""The C-ABI library loads and exports every symbol include/sparsh_b200.h
declares (no compute calls; CPU only)."""
import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "sparsh_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2007_00056_b200 import _lib
    L = _lib.lib()
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.EXPORTS)


def test_version_and_error_channel():
    from paper_2007_00056_b200 import _lib
    L = _lib.lib()
    assert b"sm_100a" in L.sb_version()
    h = ctypes.c_void_p()
    assert L.sb_setup(None, None, ctypes.byref(h)) == _lib.SB_EINVAL
    assert b"null" in L.sb_last_error()


def test_library_is_sm100a():
    import subprocess
    from paper_2007_00056_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
