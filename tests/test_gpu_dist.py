"""Partitioned (multi-rank) GPU solve on ONE device: N virtual ranks in this
process, exchanges as peer-buffer gathers (sb_dist_create_local). The
partitioned V-cycle must be bit-identical to the single-GPU V-cycle; Krylov
solves (rank-partial dots + allreduce) agree to rounding with the same
iteration counts."""
import numpy as np
import pytest

from helpers import rel

pytestmark = pytest.mark.gpu


def _cp(sp):
    return sp.CycleParams(6, 6, sp.SmootherKind.weighted_jacobi())


@pytest.mark.parametrize("nranks", [1, 2, 3, 4])
@pytest.mark.parametrize("mk,gather", [(lambda sp: sp.poisson3d(32), 4096), (lambda sp: sp.poisson2d(96, 70), 1000),
                                       (lambda sp: sp.convdiff3d(20, 18, 17, 1.0, 100.0, 1.0, 1.0), 2000)])
def test_dist_vcycle_bitexact(sp, nranks, mk, gather):
    from paper_2007_00056_b200.dist import DistSolver
    A = mk(sp)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40))
    ds = DistSolver(h, nranks, gather)
    if nranks > 1:
        assert ds.first_replicated >= 1
    f = sp.rhs_random(A.nrows(), 42)
    xd = ds.vcycle(f, _cp(sp))
    xs = sp.vcycle(h, 0, f, np.zeros(A.nrows()), _cp(sp))
    assert np.array_equal(xd, xs)


@pytest.mark.parametrize("nranks", [2, 4])
def test_dist_pcg_matches_single(sp, nranks):
    from paper_2007_00056_b200.dist import DistSolver
    A = sp.poisson3d(40)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40))
    b = sp.rhs_ones(A.nrows())
    tol = 1e-8 * np.linalg.norm(b)
    ds = DistSolver(h, nranks, 8000)
    rd = ds.pcg(b, _cp(sp), tol, 200)
    rs = sp.pcg(A, b, sp.make_amg_preconditioner(h, _cp(sp)), tol, 200)
    assert rd.report.converged() and rd.report.iterations == rs.report.iterations
    assert rel(rd.x, rs.x) < 1e-12
    assert len(rd.report.residual_history) == rd.report.iterations + 1
    assert rd.report.true_residual < 10 * tol
    assert ds.last_solve_ms() > 0


@pytest.mark.parametrize("nranks", [2, 3])
def test_dist_bicgstab_matches_single(sp, nranks):
    from paper_2007_00056_b200.dist import DistSolver
    A = sp.convdiff3d(24, 24, 24, 1.0, 100.0, 1.0, 1.0)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40))
    b = sp.rhs_ones(A.nrows())
    tol = 1e-8 * np.linalg.norm(b)
    ds = DistSolver(h, nranks, 2000)
    rd = ds.pbicgstab(b, _cp(sp), tol, 200)
    rs = sp.pbicgstab(A, b, sp.make_amg_preconditioner(h, _cp(sp)), tol, 200)
    assert rd.report.converged() and abs(rd.report.iterations - rs.report.iterations) <= 1
    assert rel(rd.x, rs.x) < 1e-9


def test_dist_identity_cg(sp):
    from paper_2007_00056_b200.dist import DistSolver
    A = sp.poisson2d(64, 64)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40))
    ds = DistSolver(h, 3, 500)
    b = sp.rhs_ones(A.nrows())
    rd = ds.pcg(b, None, 1e-300, 7)
    rs = sp.cg(A, b, 1e-300, 7)
    assert rd.report.iterations == 7 and rel(rd.x, rs.x) < 1e-12


@pytest.mark.parametrize("solver", ["pcg", "pbicgstab"])
def test_dist_nccl_one_rank_graph(sp, solver):
    """One NCCL rank: the whole distributed solve is ONE captured CUDA graph
    (NCCL calls inside conditional nodes). It must equal the eager (host-driven)
    run of the same path bit for bit, and the single-GPU solve to rounding with
    the same iteration count; the graph's kernel count equals the eager one."""
    from paper_2007_00056_b200.dist import DistSolver, nccl_unique_id
    A = sp.poisson3d(40) if solver == "pcg" else sp.convdiff3d(24, 24, 24, 1.0, 100.0, 1.0, 1.0)
    h = sp.Hierarchy(A, sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40))
    b = sp.rhs_random(A.nrows(), 3)
    tol = 1e-8 * np.linalg.norm(b)
    out = {}
    for graphs in (True, False):
        ds = DistSolver(h, 1, 4096, local=False, rank=0, nccl_id=nccl_unique_id(), graphs=graphs)
        r = getattr(ds, solver)(b, _cp(sp), tol, 200)
        r2 = getattr(ds, solver)(b, _cp(sp), tol, 200)  # graph replay
        assert np.array_equal(r.x, r2.x)
        out[graphs] = (r, ds.last_launches())
        del ds
    (rg, lg), (re, le) = out[True], out[False]
    assert rg.report.converged() and rg.report.iterations == re.report.iterations
    assert np.array_equal(rg.x.view(np.uint64), re.x.view(np.uint64))
    assert lg == le > 0
    single = getattr(sp, solver)(A, b, sp.make_amg_preconditioner(h, _cp(sp)), tol, 200)
    assert abs(single.report.iterations - rg.report.iterations) <= 1
    assert rel(rg.x, single.x) < 1e-9


# ---- peer-memory (P2P) transport -----------------------------------------------

@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("mk,gather", [(lambda sp: sp.poisson3d(32), 4096), (lambda sp: sp.poisson2d(96, 70), 1000),
                                       (lambda sp: sp.convdiff3d(20, 18, 17, 1.0, 100.0, 1.0, 1.0), 2000)])
def test_dist_p2p_vcycle_bitexact(sp, nranks, mk, gather):
    """In-process ranks over the peer-memory transport (gathers out of the peers'
    buffers, epoch flags): the partitioned V-cycle is the single-GPU one bit for bit."""
    from paper_2007_00056_b200.dist import DistSolver
    A = mk(sp)
    h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40))
    ds = DistSolver(h, nranks, gather, transport="p2p")
    f = sp.rhs_random(A.nrows(), 42)
    assert np.array_equal(ds.vcycle(f, _cp(sp)), sp.vcycle(h, 0, f, np.zeros(A.nrows()), _cp(sp)))
    assert np.array_equal(ds.vcycle(f, _cp(sp)), ds.vcycle(f, _cp(sp)))  # repeatable (epochs keep counting)


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("solver", ["pcg", "pbicgstab"])
def test_dist_p2p_solve_matches_nccl_free_local(sp, nranks, solver):
    """P2P and the event-ordered in-process transport sum the partials in the same
    rank order: the solves agree bit for bit; both match the single-GPU solve."""
    from paper_2007_00056_b200.dist import DistSolver
    A = sp.poisson3d(32) if solver == "pcg" else sp.convdiff3d(20, 18, 17, 1.0, 100.0, 1.0, 1.0)
    h = sp.Hierarchy(A, sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40))
    b = sp.rhs_random(A.nrows(), 9)
    tol = 1e-8 * np.linalg.norm(b)
    rp = getattr(DistSolver(h, nranks, 2048, transport="p2p"), solver)(b, _cp(sp), tol, 200)
    rl = getattr(DistSolver(h, nranks, 2048), solver)(b, _cp(sp), tol, 200)
    assert rp.report.converged() and rp.report.iterations == rl.report.iterations
    assert np.array_equal(rp.x.view(np.uint64), rl.x.view(np.uint64))
    single = getattr(sp, solver)(A, b, sp.make_amg_preconditioner(h, _cp(sp)), tol, 200)
    assert abs(single.report.iterations - rp.report.iterations) <= 1
    assert rel(rp.x, single.x) < 1e-9


_P2P_WORKER = r"""
import os, sys, time, json, numpy as np
sys.path.insert(0, os.environ["SB_ROOT"])
from paper_2007_00056_b200 import sparsh as sp
from paper_2007_00056_b200.dist import DistSolver
rank, nranks, tmp, graphs = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4] == "1"
A = sp.poisson3d(28)
h = sp.Hierarchy(A, sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40))
ds = DistSolver(h, nranks, 2048, local=False, rank=rank, transport="p2p", graphs=graphs)
open(os.path.join(tmp, f"blob{rank}.tmp"), "wb").write(ds.p2p_export())
os.replace(os.path.join(tmp, f"blob{rank}.tmp"), os.path.join(tmp, f"blob{rank}"))
while not all(os.path.exists(os.path.join(tmp, f"blob{q}")) for q in range(nranks)):
    time.sleep(0.05)
ds.p2p_connect([open(os.path.join(tmp, f"blob{q}"), "rb").read() for q in range(nranks)])
b = sp.rhs_ones(A.nrows())[ds.lo:ds.hi]
cp = sp.CycleParams(6, 6, sp.SmootherKind.weighted_jacobi())
tol = 1e-8 * np.sqrt(A.nrows())
r1 = ds.pcg(b, cp, tol, 100)
r2 = ds.pcg(b, cp, tol, 100)  # graph replay / second eager run
assert np.array_equal(r1.x, r2.x)
np.save(os.path.join(tmp, f"x{rank}.npy"), r1.x)
json.dump({"it": r1.report.iterations, "lo": ds.lo, "hi": ds.hi}, open(os.path.join(tmp, f"r{rank}.json"), "w"))
"""


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_dist_p2p_two_processes_ipc(sp, tmp_path, graphs):
    """Two PROCESSES (one rank each) on the same GPU over CUDA IPC: each exports
    its buffers, connects to the other's, and solves (as one captured graph, or
    eagerly); the joined solution equals the in-process P2P solve bit for bit."""
    import json
    import os
    import subprocess
    import sys
    from conftest import ROOT
    from paper_2007_00056_b200.dist import DistSolver
    script = tmp_path / "w.py"
    script.write_text(_P2P_WORKER)
    env = dict(os.environ, SB_ROOT=ROOT)
    procs = [subprocess.Popen([sys.executable, str(script), str(r), "2", str(tmp_path), graphs], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    A = sp.poisson3d(28)
    h = sp.Hierarchy(A, sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40))
    ref = DistSolver(h, 2, 2048, transport="p2p").pcg(sp.rhs_ones(A.nrows()), _cp(sp), 1e-8 * np.sqrt(A.nrows()), 100)
    x = np.zeros(A.nrows())
    for r in range(2):
        m = json.load(open(tmp_path / f"r{r}.json"))
        assert m["it"] == ref.report.iterations
        x[m["lo"]:m["hi"]] = np.load(tmp_path / f"x{r}.npy")
    assert np.array_equal(x.view(np.uint64), ref.x.view(np.uint64))


_OVERLAP_WORKER = r"""
import os, sys, json, hashlib, numpy as np
sys.path.insert(0, os.environ["SB_ROOT"])
from paper_2007_00056_b200 import sparsh as sp
from paper_2007_00056_b200.dist import DistSolver
A = sp.poisson3d(48)
h = sp.Hierarchy(A, sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40))
cp = sp.CycleParams(6, 6, sp.SmootherKind.weighted_jacobi())
b = sp.rhs_ones(A.nrows())
out = {}
for transport in ("local", "p2p"):
    for graphs in (True, False):
        ds = DistSolver(h, 2, 2048, transport=transport, graphs=graphs)
        r = ds.pcg(b, cp, 1e-8 * np.sqrt(A.nrows()), 100)
        out[f"{transport}-{int(graphs)}"] = [r.report.iterations, ds.last_launches(),
                                             hashlib.sha1(r.x.tobytes()).hexdigest()]
print(json.dumps(out))
"""


def test_dist_interior_overlap_bitwise():
    """The halo/interior overlap (interior row pairs swept while the halo is in
    flight, then the edge rows) changes the launch sequence, not one bit of the
    solution: on vs off (SB_DIST_OVERLAP=0), both transports, graph and eager."""
    import json
    import os
    import subprocess
    import sys
    from conftest import ROOT
    res = {}
    for ov in ("1", "0"):
        env = dict(os.environ, SB_ROOT=ROOT, SB_DIST_OVERLAP=ov)
        p = subprocess.run([sys.executable, "-c", _OVERLAP_WORKER], env=env, capture_output=True, text=True,
                           timeout=600)
        assert p.returncode == 0, p.stderr[-3000:]
        res[ov] = json.loads(p.stdout.strip().splitlines()[-1])
    hashes = {v[2] for r in res.values() for v in r.values()}
    assert len(hashes) == 1, res
    for key in res["1"]:
        assert res["1"][key][0] == res["0"][key][0]
    # overlap active on the P2P transport (publish / interior / wait / edges)
    # and on the eager local transport (side stream)
    assert res["1"]["p2p-1"][1] > res["0"]["p2p-1"][1], res
    assert res["1"]["local-0"][1] > res["0"]["local-0"][1], res
