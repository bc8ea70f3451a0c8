"""The command-line front end (paper_2007_00056_b200/_lib/sparsh_b200), the
`sparsh run / gen / coarsen-info` equivalent (tools/sparsh.cpp), re-expressing
tests/test_cli.cpp of the reference: gen writes the reference's Matrix Market
text, run writes the convergence CSV (first residual ||b||, iter column counting
up, timing non-decreasing), runs are deterministic, a matrix file reproduces the
generated problem, unconverged runs exit 1, usage errors exit 2."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CLI = os.path.join(ROOT, "paper_2007_00056_b200", "_lib", "sparsh_b200")


def run_cli(*args, cwd=None):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300, cwd=cwd)
    return r.returncode, r.stdout, r.stderr


def rows(csv_text):
    lines = [l for l in csv_text.splitlines() if l]
    assert lines[0] == "iter,residual_l2,cumulative_seconds"
    return [l.rsplit(",", 1) for l in lines[1:]]


def test_gen_matches_reference_writer(sp, ref, tmp_path):
    out = tmp_path / "m.mtx"
    code, _, err = run_cli("gen", "--problem", "poisson2d:3x3", "--out", out)
    assert code == 0, err
    theirs = tmp_path / "ref.mtx"
    ref.write_matrix_market(sp.poisson2d(3, 3), theirs)
    assert out.read_text() == theirs.read_text()
    code, text, _ = run_cli("gen", "--problem", "poisson2d:3x3")  # stdout by default
    assert code == 0 and text == theirs.read_text()


def test_coarsen_info_matches_hierarchy(sp):
    code, out, err = run_cli("coarsen-info", "--problem", "poisson2d:32x32", "--max-levels", "3",
                             "--coarse-target", "1")
    assert code == 0, err
    sizes = [int(l.split()[1]) for l in out.splitlines()[1:4]]
    assert sizes == [1024, 512, 256]  # test_hierarchy.cpp:60-68
    assert "operator complexity:" in out and "grid complexity:" in out


@pytest.mark.parametrize("args,msg", [
    (["run"], "exactly one of --problem and --matrix"),
    (["run", "--problem", "poisson2d:4"], "bad --problem"),
    (["run", "--problem", "poisson2d:8x8", "--rhs", "zeros"], "bad --rhs"),
    (["run", "--problem", "poisson2d:8x8", "--bogus", "1"], "unknown option --bogus"),
    (["run", "--problem", "poisson2d:8x8", "--smoother", "gs_symmetric"], "Gauss-Seidel"),
    (["run", "--matrix", "/nonexistent.mtx"], "cannot open"),
])
def test_usage_errors_exit_2(args, msg):
    code, _, err = run_cli(*args)
    assert code == 2 and msg in err, (code, err)


@pytest.mark.gpu
def test_run_writes_report_csv(tmp_path):
    csv = tmp_path / "r.csv"
    code, out, err = run_cli("run", "--problem", "poisson2d:16x16", "--solver", "pcg", "--out", csv)
    assert code == 0, err
    assert "termination: converged" in out and "solver: pcg" in out
    rs = rows(csv.read_text())
    assert len(rs) >= 2 and rs[0][0] == "0,16"  # ||b|| = sqrt(256) (test_cli.cpp:117-119)
    assert float(rs[-1][0].split(",")[1]) < 1e-8
    iters = [int(r[0].split(",")[0]) for r in rs]
    assert iters == list(range(len(rs)))
    secs = [float(r[1]) for r in rs]
    assert all(b >= a for a, b in zip(secs, secs[1:]))


@pytest.mark.gpu
def test_run_matches_oracle_iterations(sp, oracle_best):
    code, out, err = run_cli("run", "--problem", "poisson2d:64x64", "--solver", "pcg", "--max-levels", "40")
    assert code == 0, err
    it = int([l for l in out.splitlines() if l.startswith("iterations:")][0].split()[1])
    A = sp.poisson2d(64, 64)
    o = oracle_best.hierarchy(A, 500, 40)
    assert abs(it - o.pcg(np.ones(A.nrows()), 1e-8, 1000).iterations) <= 1


@pytest.mark.gpu
def test_run_deterministic_and_matrix_file_reproduces(tmp_path):
    mtx, a, b, c = tmp_path / "m.mtx", tmp_path / "a.csv", tmp_path / "b.csv", tmp_path / "c.csv"
    assert run_cli("gen", "--problem", "poisson2d:16x16", "--out", mtx)[0] == 0
    for f in (a, b):
        assert run_cli("run", "--problem", "poisson2d:16x16", "--solver", "amg", "--out", f)[0] == 0
    assert run_cli("run", "--matrix", mtx, "--solver", "amg", "--out", c)[0] == 0
    strip = lambda p: [r[0] for r in rows(p.read_text())]  # noqa: E731  (timing column varies)
    assert strip(a) == strip(b) == strip(c)


@pytest.mark.gpu
@pytest.mark.parametrize("solver,problem", [("cg", "poisson2d:24x24"), ("bicgstab", "convdiff2d:24x24:1,100,1"),
                                            ("pbicgstab", "convdiff2d:24x24:1,100,1")])
def test_run_other_solvers(solver, problem):
    code, out, err = run_cli("run", "--problem", problem, "--solver", solver, "--max-levels", "40")
    assert code == 0, err
    assert f"solver: {solver}" in out and "termination: converged" in out


@pytest.mark.gpu
def test_unconverged_run_exits_1(tmp_path):
    code, out, err = run_cli("run", "--problem", "poisson2d:32x32", "--solver", "pcg", "--max-iters", "2",
                             "--tol", "1e-14", "--out", tmp_path / "r.csv")
    assert code == 1 and "did not converge" in err and "termination: max_iters" in out
