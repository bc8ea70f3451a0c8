"""The header-only C++ drop-in (include/sparsh_b200.hpp) compiles against the
C ABI and runs a reference-style program (tests/cpp/drop_in.cpp) on the GPU."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_drop_in(tmp_path):
    exe = tmp_path / "drop_in"
    lib = os.path.join(ROOT, "paper_2007_00056_b200", "_lib")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "drop_in.cpp"), "-L", lib, "-lsparsh_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["pcg_converged"] == 1 and d["gs_rejected"] == 1 and d["hybrid_same"] == 1
    assert 5 <= d["pcg_iters"] <= 20 and d["cg_iters"] > d["pcg_iters"]
    assert d["true_residual"] < 1e-6


def test_cpp_header_compiles_without_cuda_headers(tmp_path):
    # the C ABI header is plain C: no CUDA / torch types cross the boundary
    src = tmp_path / "c_only.c"
    src.write_text('#include "sparsh_b200.h"\nint main(void){ return sb_version() ? 0 : 1; }\n')
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-c", str(src), "-o",
                    str(tmp_path / "c_only.o")], check=True)
