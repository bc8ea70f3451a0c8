"""Multi-rank (world size 2 and 3, gloo on CPU) check of the row partition and
its exchange plans (sb_partition*): a distributed V-cycle and SpMV executed in
numpy with the plans and real torch.distributed send/recv must reproduce the
global computation BIT FOR BIT (row sums keep CSR order; restriction and
prolongation are exact), and dot products must agree to rounding."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

OMEGA = 2.0 / 3.0


def rowsum(A, x):
    """y_i = sum_k a_k x_{c_k} sequentially in CSR order (the reference's spmv)."""
    rp = A.row_ptr().astype(np.int64)
    ln = np.diff(rp)
    y = np.zeros(A.nrows())
    for k in range(int(ln.max()) if ln.size else 0):
        m = ln > k
        idx = rp[:-1][m] + k
        y[m] = y[m] + A.values()[idx] * x[A.col_idx()[idx]]
    return y


def diag_of(A, ncol_own=None):
    rp = A.row_ptr().astype(np.int64)
    d = np.zeros(A.nrows())
    for i in range(A.nrows()):
        for k in range(rp[i], rp[i + 1]):
            if A.col_idx()[k] == i:
                d[i] = A.values()[k]
    return d


def jacobi(A, d, x, f, x_is_zero):
    if x_is_zero:
        return 0.0 + (OMEGA * (f - 0.0)) / d
    return x + (OMEGA * (f - rowsum(A, x))) / d


def vcycle_global(levels, k, f, pre, post, coarse):
    A = levels[k].A
    if k + 1 == len(levels):
        return coarse(f)
    d = diag_of(A)
    x = None
    for s in range(pre):
        x = jacobi(A, d, x, f, s == 0)
    if pre == 0:
        x = np.zeros(A.nrows())
    r = f - rowsum(A, x)
    agg = levels[k].agg.fine_to_coarse
    fc = np.zeros(levels[k].agg.n_coarse)
    for i in range(A.nrows()):
        fc[agg[i]] += 1.0 * r[i]
    xc = vcycle_global(levels, k + 1, fc, pre, post, coarse)
    x = x + (0.0 + xc[agg])
    for s in range(post):
        x = jacobi(A, d, x, f, False)
    return x


def exchange(plan, own, tag):
    """Fill the ghost values for this rank from `own` of every peer (gloo)."""
    reqs, out = [], np.zeros(int(plan["recv_off"][-1]) if len(plan["recv_off"]) else 0)
    import torch
    bufs = []
    for i, q in enumerate(plan["send_peers"]):
        seg = own[plan["send_idx"][plan["send_off"][i]:plan["send_off"][i + 1]]]
        t = torch.from_numpy(np.ascontiguousarray(seg))
        bufs.append(t)
        reqs.append(dist.isend(t, int(q), tag=tag))
    rbufs = []
    for i, q in enumerate(plan["recv_peers"]):
        t = torch.zeros(int(plan["recv_off"][i + 1] - plan["recv_off"][i]), dtype=torch.float64)
        rbufs.append((i, t))
        reqs.append(dist.irecv(t, int(q), tag=tag))
    for r in reqs:
        r.wait()
    for i, t in rbufs:
        out[plan["recv_off"][i]:plan["recv_off"][i + 1]] = t.numpy()
    return out


def halo_ext(pl, plan, v, tag):
    """x vector of a partitioned level with its halo: [wb rows below | own | wa rows
    above]; each peer's chunk lands at wb + recv_dst (window layout: ghosts at
    their global offsets; compact layout: wb = 0, ghosts packed after own)."""
    wb, wa, n = int(pl["wb"]), int(pl["wa"]), v.size
    xe = np.zeros(wb + n + wa)
    xe[wb:wb + n] = v
    g = exchange(plan, v, tag)
    for j in range(len(plan["recv_peers"])):
        a, b = int(plan["recv_off"][j]), int(plan["recv_off"][j + 1])
        d = wb + int(plan["recv_dst"][j])
        xe[d:d + (b - a)] = g[a:b]
    return xe


def shifted(sp, pl):
    """the local matrix with columns indexing halo_ext()'s vector"""
    A = pl["A"]
    return sp.CsrMatrix(A.nrows(), int(pl["wb"]) + A.nrows() + int(pl["wa"]), A.row_ptr(),
                        A.col_idx() + int(pl["wb"]), A.values(), _validate=False)


def vcycle_dist(part, levels, k, f_own, pre, post, coarse, tagbase):
    pl = part.level(k)
    if pl["replicated"]:
        return vcycle_global(levels, k, f_own, pre, post, coarse)
    from paper_2007_00056_b200 import sparsh as sp
    A = shifted(sp, pl)  # columns index the halo-extended vector
    n = A.nrows()
    d = diag_of(pl["A"])
    halo = part.exchange(k, 0)
    tag = [tagbase]

    def ext(v):
        tag[0] += 1
        return halo_ext(pl, halo, v, tag[0])

    x = np.zeros(n)
    for s in range(pre):
        if s == 0:
            x = 0.0 + (OMEGA * (f_own - 0.0)) / d  # first sweep from x = 0
        else:
            xe = ext(x)
            x = x + (OMEGA * (f_own - rowsum(A, xe))) / d
    r = f_own - rowsum(A, ext(x))
    tag[0] += 1
    r_ext = np.concatenate([r, exchange(part.exchange(k, 1), r, tag[0])])
    fc = np.array([(0.0 + r_ext[a]) + (r_ext[b] if b >= 0 else 0.0) if b >= 0 else 0.0 + r_ext[a]
                   for a, b in zip(pl["mem0"], pl["mem1"])])
    nxt = part.level(k + 1) if k + 1 < part.nlevels else None
    if nxt["replicated"]:
        pieces = [None] * part.nranks
        dist.all_gather_object(pieces, fc)
        fc_full = np.concatenate(pieces)
        xc = vcycle_global(levels, k + 1, fc_full, pre, post, coarse)
        x = x + (0.0 + xc[pl["parent"]])
    else:
        xc = vcycle_dist(part, levels, k + 1, fc, pre, post, coarse, tag[0] + 1000)
        tag[0] += 2000
        xc_ext = np.concatenate([xc, exchange(part.exchange(k, 2), xc, tag[0])])
        x = x + (0.0 + xc_ext[pl["parent"]])
    for s in range(post):
        xe = ext(x)
        x = x + (OMEGA * (f_own - rowsum(A, xe))) / d
    return x


def _worker(rank, ws, port, results):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2007_00056_b200 import sparsh as sp
        from paper_2007_00056_b200.dist import Partition
        stats = []
        for mk, gather in [(lambda: sp.poisson3d(16), 512), (lambda: sp.poisson2d(40, 33), 200),
                           (lambda: sp.convdiff3d(12, 10, 9, 1.0, 100.0, 1.0, 1.0), 300)]:
            A = mk()
            h = sp.Hierarchy(A, sp.SolverConfig(max_levels=40, coarse_target=64))
            levels = h.levels()
            Ac = levels[-1].A.to_dense()
            coarse = lambda f: np.linalg.solve(Ac, f)  # noqa: E731  (same inputs on every rank)
            part = Partition(h, rank, ws, gather)
            assert part.first_replicated >= 1
            f = sp.rhs_random(A.nrows(), 42)
            lo, hi = part.level(0)["lo"], part.level(0)["hi"]
            xg = vcycle_global(levels, 0, f, 6, 6, coarse)
            xd = vcycle_dist(part, levels, 0, f[lo:hi], 6, 6, coarse, 1)
            assert np.array_equal(xd, xg[lo:hi]), (rank, np.abs(xd - xg[lo:hi]).max())
            straddle = sum(len(part.level(k)["rghost"]) + len(part.level(k)["xcghost"])
                           for k in range(part.first_replicated))
            stats.append(straddle)
            # distributed SpMV + allreduced dot
            import torch
            pl = part.level(0)
            xe = halo_ext(pl, part.exchange(0, 0), f[lo:hi], 99999)
            y = rowsum(shifted(sp, pl), xe)
            assert np.array_equal(y, rowsum(A, f)[lo:hi])
            t = torch.tensor([float(np.dot(y, f[lo:hi]))], dtype=torch.float64)
            dist.all_reduce(t)
            assert abs(t.item() - float(np.dot(rowsum(A, f), f))) <= 1e-12 * abs(t.item())
        results[rank] = "ok"
        results[f"straddle{rank}"] = sum(stats)
    except Exception as e:  # report to the parent
        import traceback
        results[rank] = traceback.format_exc()
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ws", [2, 3])
def test_partitioned_vcycle_bitexact_gloo(ws):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, results)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    for r in range(ws):
        assert results.get(r) == "ok", results.get(r)
    # the uneven row split creates aggregates straddling ranks: their
    # residual / coarse-parent exchanges were exercised
    assert sum(results.get(f"straddle{r}", 0) for r in range(ws)) > 0
