#!/usr/bin/env python
"""Benchmark: AMG-PCG solve of BASELINE.json configs[1] (C2: 3D 7-point Poisson
128^3, 2.1M DOFs, Jacobi 6/6, node-HEM, coarse_target 500, max_levels 40,
rhs = ones, tol = 1e-8 * ||b||) on N GPUs of one node. One "step" = one full
PCG solve to tolerance.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload C2|C1|C3|C4]

`value`  = device time of one solve (CUDA events on the solve stream, inputs
           resident in HBM; L2 flushed before every step), max over ranks.
`e2e`    = the same solve through the public C ABI with host (pinned) b and x:
           H2D of b, solve, D2H of x inside the timed region.
`roofline` = the L0 Jacobi sweep kernel k_sellg<JACOBI> (the dominant kernel),
           algorithmic bytes / CUDA-event duration vs MEASURED_PEAKS.json.
`cpu_baseline` = the reference's own CPU code (oracle/_ref) on this host.
N > 1 (torchrun): the row-partitioned solve (sb_dist_*: NCCL halo exchanges and
dot-product allreduces); default workload = C2 weak-scaled (128 x 128 x 128N
grid, z-slab row blocks) -> `scaling: weak`; --workload C3/C4 = strong scaling.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AMG-PCG solve s to 1e-8 rel. residual; SpMV/V-cycle HBM GB/s vs peak, 1–8 GPU"

WORKLOADS = {
    "C2": dict(desc="C2: 3D 7-pt Poisson 128^3 (2.1M DOFs) AMG-PCG, full hierarchy device-resident",
               solver="pcg", gen=lambda sp: sp.poisson3d(128)),
    "C1": dict(desc="C1: 2D 5-pt Poisson 1024^2 (1M DOFs) AMG-PCG",
               solver="pcg", gen=lambda sp: sp.poisson2d(1024, 1024)),
    "C3": dict(desc="C3: 3D anisotropic (eps=1e-3 in z) 7-pt 256^3 (16.8M DOFs) AMG-PCG",
               solver="pcg", gen=lambda sp: sp.aniso3d(256, 1e-3)),
    "C4": dict(desc="C4: 3D convection-diffusion 256^3, b=(1,100,1), c=1 AMG-PBiCGStab",
               solver="pbicgstab", gen=lambda sp: sp.convdiff3d(256, 256, 256, 1.0, 100.0, 1.0, 1.0)),
    # BASELINE.json's stated target: "3D 7-point Poisson 256^3 AMG-PCG solved to 1e-8"
    "T256": dict(desc="Target: 3D 7-pt Poisson 256^3 (16.8M DOFs) AMG-PCG to 1e-8",
                 solver="pcg", gen=lambda sp: sp.poisson3d(256)),
    # a general-valued operator (every row distinct, irregular coarse levels):
    # the SELL-G / CSR format path instead of the row-pattern one
    "G128": dict(desc="G128: 3D 7-pt graph Laplacian 128^3, random edge weights U[0.5,1.5) + 0.01 I (general "
                      "format path) AMG-PCG",
                 solver="pcg", gen=lambda sp: sp.graph_laplacian3d(128, seed=7)),
}



def placement(h, args):
    """Level placement of the run: all levels device-resident, or the paper's hybrid
    scheme (levels >= host_levels_from in pinned host memory, read zero-copy)."""
    if args.host_levels_from < 0:
        return {"mode": "device", "device_gb": round(h.device_bytes() / 1e9, 3)}
    return {"mode": "hybrid", "host_levels_from": args.host_levels_from,
            "device_gb": round(h.device_bytes() / 1e9, 3), "host_gb": round(h.host_bytes() / 1e9, 3)}


def run_c5(args, wl):
    """C5 (BASELINE configs[4]): 3D 27-point Poisson 512^3 (134M DOFs, nnz 3.6e9 > int32)
    AMG-PCG on ONE GPU (the config names 8 GPUs + hybrid; one B200 holds the whole
    hierarchy in row-pattern form). The operator is generated straight into the
    setup (sb_setup_stencil27: no Python copy of the 44 GB fine matrix). The
    reference cannot build this system (int32 offsets), so there is no CPU arm;
    parity is pinned on the 27-point proxies the reference can run (tests)."""
    import ctypes as C
    import torch
    from paper_2007_00056_b200 import sparsh as sp, _lib
    nside = 512 if wl == "C5" else 256
    L = _lib.lib()
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40, coarse_target=500)
    t0 = time.perf_counter()
    h = sp.Hierarchy.from_stencil27(nside, nside, nside, 26.0, -1.0, cfg, galerkin_gpu=args.galerkin_gpu,
                                    host_levels_from=args.host_levels_from)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    ctx = h.ctx()
    t_upload = time.perf_counter() - t0
    lv = []
    for k in range(h.nlevels()):
        a = _lib.sb_csr()
        agg = C.POINTER(C.c_int32)()
        nc = C.c_int64()
        _lib.check(L.sb_hier_level(h._h, k, C.byref(a), C.byref(agg), C.byref(nc)))
        nnz = a.row_ptr64[a.nrows] if a.row_ptr64 else a.row_ptr32[a.nrows]
        fmt = (C.c_int * 4)()
        mb, nz = C.c_int64(), C.c_int64()
        _lib.check(L.sb_level_format(ctx, k, fmt, C.byref(mb), C.byref(nz)))
        lv.append((a.nrows, int(nnz), mb.value, list(fmt)))
    n = lv[0][0]
    cp = sp.CycleParams.from_config(cfg)._abi()
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    tol = 1e-8 * float(np.sqrt(n))
    rep = _lib.sb_report()

    def solve():
        _lib.check(L.sb_pcg_dev(ctx, C.byref(cp), C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), tol, 1000,
                                C.byref(rep)))
        return rep

    for _ in range(max(args.warmup, 3)):
        solve()
    assert rep.termination == 0, f"C5 solve did not converge: {rep.termination}"
    per = []
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            solve()
            per.append(L.sb_last_solve_ms(ctx))
        torch.cuda.synchronize()
    ms = statistics.mean(per)
    avg, cnt = C.c_double(), C.c_int()
    _lib.check(L.sb_time_kernel(ctx, 0, 0, C.byref(cp), 10, C.byref(avg), C.byref(cnt)))
    jac_bytes = lv[0][2] + 24 * n
    peak, peak_kind = peaks()
    achieved = jac_bytes / (avg.value * 1e-3) / 1e9
    b_pin = torch.ones(n, dtype=torch.float64).pin_memory()
    x_pin = torch.zeros(n, dtype=torch.float64).pin_memory()
    bp = C.cast(C.c_void_p(b_pin.data_ptr()), C.POINTER(C.c_double))
    xp = C.cast(C.c_void_p(x_pin.data_ptr()), C.POINTER(C.c_double))
    e2e = []
    for i in range(1 + min(args.steps, 3)):
        rep2 = _lib.sb_report()
        t1 = time.perf_counter()
        _lib.check(L.sb_pcg(ctx, C.byref(cp), bp, xp, tol, 1000, C.byref(rep2)))
        if i:
            e2e.append(time.perf_counter() - t1)
    line = {"metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"C5: 3D 27-pt Poisson {nside}^3 ({n} DOFs, nnz {lv[0][1]}) AMG-PCG on 1 GPU "
                                   f"(row-pattern storage: {h.device_bytes() / 1e9:.1f} GB device-resident)",
                       "n": n, "nnz": lv[0][1], "levels": len(lv), "iterations": rep.iterations, "rhs": "ones",
                       "tol": "1e-8*||b||", "true_rel_residual": rep.true_residual / float(np.sqrt(n)),
                       "setup_s": round(t_setup, 1), "upload_s": round(t_upload, 1),
                       "level_rows": [v[0] for v in lv], "level_formats": [v[3][0] for v in lv],
                       "placement": placement(h, args), "parallelism": "single GPU"},
            "roofline": {"bound": "hbm", "kernel": sweep_kernel(L, ctx) + " (L0 Jacobi sweep)", "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "frac_of_spec_8000": achieved / SPEC_HBM_GBS,
                         # C5p's operator is the 27-point 256^3 of profiles/ncu_summary_P27_256.json
                         "traffic": load_traffic("P27_256") if wl == "C5p" else None,
                         "algorithmic_bytes_per_launch": jac_bytes, "launch_ms": avg.value},
            "e2e": {"value": statistics.mean(e2e), "unit": "s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n},
            "cpu_baseline": {"value": None, "unit": "s", "cores": 0, "kind": "reference",
                             "sample": "unavailable: the reference's int32 CSR offsets cannot hold nnz = 3.6e9"},
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


SPEC_HBM_GBS = 8000.0  # BASELINE.json's "~8 TB/s per-GPU peak" (report both)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(s[0]) for s in self.samples if num(s[0])]
        busy = [num(s[0]) for s in self.samples if num(s[0]) and (num(s[6]) or 0) > 0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(num(s[1]) or 0 for s in self.samples), "reasons": reasons,
                "samples": len(self.samples)}


def bytes_model(h, pre=6, post=6, matrix_bytes=None):
    """Algorithmic bytes: the matrix once per pass, each distinct
    vector once. matrix_bytes[k] = bytes one pass over level k's matrix streams;
    None = the survey's CSR figure 12 B/nnz + 4 B/row offset. With the shipped
    lossless format (value dictionary, int16 column deltas, sliced ELL) pass
    sb_level_format's matrix bytes instead."""
    lv = [(l.A.nrows(), l.A.nnz()) for l in h.levels()]
    L = len(lv)
    M = matrix_bytes or [12 * z + 4 * (n + 1) for n, z in lv]

    def jac(k):
        return M[k] + 24 * lv[k][0]

    vc = 0
    for k in range(L - 1):
        n, z = lv[k]
        nc = lv[k + 1][0]
        vc += (pre + post - 1) * jac(k) + 24 * n                   # sweeps + zero-guess sweep
        vc += M[k] + 16 * n + 4 * n + 8 * nc                       # residual + restriction
        vc += 16 * n + 4 * n + 8 * nc                              # prolongation
    ncs = lv[-1][0]
    vc += 8 * ncs * ncs + 16 * ncs
    n0 = lv[0][0]
    spmv = M[0] + 16 * n0
    pcg_it = vc + spmv + 40 * n0 + 16 * n0 + 24 * n0
    # BiCGStab (krylov.hpp:156-205 as fused here): 2 V-cycles; 2 SpMVs with their dots
    # (A pt, (A pt, rbar); A st, (As, As), (As, s)) = 2 M + 48 n; s = r - a Apt (+||s||) 24 n;
    # x, r update (+2 dots) 64 n; p = r + b (p - w Apt) 32 n
    bicg_it = 2 * vc + 2 * M[0] + 48 * n0 + 24 * n0 + 64 * n0 + 32 * n0
    return dict(vcycle=vc, pcg_iter=pcg_it, bicg_iter=bicg_it, l0_jacobi=jac(0), l0_spmv=spmv)


def sweep_kernel(L, ctx, level=0):
    """The kernel a Jacobi sweep of `level` launches (sb_level_sweep_kernel)."""
    import ctypes as C
    buf = C.create_string_buffer(64)
    from paper_2007_00056_b200 import _lib
    _lib.check(L.sb_level_sweep_kernel(ctx, level, buf, 64))
    return buf.value.decode() + "<JACOBI>"
def bytes_of_format(fmt):
    """What one matrix pass streams for a level format (sb_level_format: kind, vf, cf, width)."""
    kind, vf, cf = fmt[0], fmt[1], fmt[2]
    v = "1 B value index" if vf else "8 B value"
    c = "2 B column delta" if cf else "4 B column"
    if kind == 2:
        return "matrix pass = 1 B pattern index per row + the pattern table"
    if kind == 1:
        return (f"matrix pass = grouped sliced-ELL slice blocks incl. padding ({v} + {c} per slot, "
                "2 B/row length + diagonal index, 16 B/slice header)")
    return f"matrix pass = CSR tiles ({v} + {c} per nonzero + 4 B/row)"


def load_traffic(wl):
    """dram read+write bytes of one L0 Jacobi sweep launch from the committed ncu
    capture of THIS workload (profiles/ncu_summary[_WL].json), else None."""
    name = "ncu_summary.json" if wl == "C2" else f"ncu_summary_{wl}.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f).get("jacobi_l0_dram_bytes_per_launch")
    except Exception:
        return None


def run_reference(args, wl):
    """--impl reference: the reference's own CPU code (oracle/_ref: the unmodified
    sparsh headers compiled by oracle/Makefile) on this host's cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    from paper_2007_00056_b200 import sparsh as sp  # generator only (same matrix as our arm)
    try:
        R = orc.Ref()
        kind = "reference"
    except Exception:
        R = orc.Port()
        kind = "port"
    cores = os.cpu_count() or 1
    if kind == "reference":
        R.set_threads(cores)
    A = WORKLOADS[wl]["gen"](sp)
    b = sp.rhs_ones(A.nrows())
    tol = 1e-8 * float(np.linalg.norm(b))
    h = R.hierarchy(A, 500, 40)
    solver = WORKLOADS[wl]["solver"]
    k_full = REF_ITERS.get(wl, REF_ITERS_MEASURED.get(wl))
    m = args.ref_sample_iters
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = getattr(h, solver)(b, tol, m)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = statistics.median(times)
    # full solve with k iterations ~ (k + 1) preconditioner applications; the
    # m-iteration sample performs m + 1 (krylov.hpp:85,109) -> scale by (k+1)/(m+1)
    scale = (k_full + 1) / (m + 1) if solver == "pcg" else k_full / m
    value = t * scale
    line = {"metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOADS[wl]["desc"], "n": A.nrows(), "nnz": A.nnz(),
                       "tol": "1e-8*||b||", "rhs": "ones", "parallelism": "cpu-threads"},
            "cpu_baseline": {"value": value, "unit": "s", "cores": cores if kind == "reference" else 1,
                             "kind": kind,
                             "sample": f"{solver} max_iters={m} on the full {wl} system per step "
                                       f"(median {t:.3f} s), scaled x{scale:.2f} to the {k_full}-iteration "
                                       f"solve"},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# iteration counts of the reference at these configs (re-checked by tests)
REF_ITERS = {"C1": 60, "C2": 22, "C3": 43, "C4": 20}
# iteration counts the GPU path measured (bitwise-parity tests pin it to the reference's)
REF_ITERS_MEASURED = {"T256": 32}


def cpu_baseline_sample(A, b, tol, wl, sample_iters, gpu_iters=None):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    try:
        R = orc.Ref()
        kind = "reference"
    except Exception:
        R = orc.Port()
        kind = "port"
    cores = os.cpu_count() or 1
    if kind == "reference":
        R.set_threads(cores)
    h = R.hierarchy(A, 500, 40)
    solver = WORKLOADS[wl]["solver"]
    t0 = time.perf_counter()
    getattr(h, solver)(b, tol, sample_iters)
    dt = time.perf_counter() - t0
    k = REF_ITERS.get(wl, gpu_iters)  # same iteration count as the reference (parity tests)
    scale = (k + 1) / (sample_iters + 1) if solver == "pcg" else k / sample_iters
    return {"value": dt * scale, "unit": "s", "cores": cores if kind == "reference" else 1, "kind": kind,
            "sample": f"{solver} max_iters={sample_iters} on the full {wl} system ({dt:.2f} s), "
                      f"scaled x{scale:.2f} to the {k}-iteration solve"}


def run_multi(args, wl):
    """N > 1 GPUs (torchrun, one rank per GPU): the row-partitioned solve
    (libsparsh_b200 sb_dist_*, NCCL halo exchanges / allreduce; levels below
    --gather-rows replicated). Default workload: weak scaling of C2 — the
    7-pt Poisson grid 128 x 128 x (128 N), z-slab row blocks, so N = 1 is C2
    itself. --workload C3/C4/C1: strong scaling of that config."""
    import torch
    import torch.distributed as dist
    from paper_2007_00056_b200 import sparsh as sp
    from paper_2007_00056_b200.dist import DistSolver, nccl_unique_id

    ws, rank, local = dist_env()
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    if wl == "C2":
        A = sp.poisson3d(128, 128, 128 * ws)
        desc = f"C2 weak-scaled: 3D 7-pt Poisson 128x128x{128 * ws} ({A.nrows() // ws} DOFs per GPU) AMG-PCG, row-partitioned"
        scaling = "weak"
    else:
        A = WORKLOADS[wl]["gen"](sp)
        desc = WORKLOADS[wl]["desc"] + f", row-partitioned over {ws} GPUs"
        scaling = "strong"
    n = A.nrows()
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40, coarse_target=500)
    t0 = time.perf_counter()
    h = sp.Hierarchy(A, cfg, device=local)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ds = DistSolver(h, ws, args.gather_rows, local=False, rank=rank, nccl_id=obj[0], device=local)
    setup_s = time.perf_counter() - t0
    cp = sp.CycleParams.from_config(cfg)
    solver = WORKLOADS[wl]["solver"]
    nloc = ds.hi - ds.lo
    tol = 1e-8 * float(np.sqrt(n))  # ||ones(n)||
    fn = ds.pcg if solver == "pcg" else ds.pbicgstab
    b_dev = torch.ones(nloc, dtype=torch.float64, device=f"cuda:{local}")
    x_dev = torch.zeros(nloc, dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    for _ in range(max(args.warmup, 3)):
        rep = fn(b_dev.data_ptr(), cp, tol, 1000, x_dev.data_ptr()).report
    assert rep.converged(), f"multi-GPU solve did not converge: {rep.termination}"
    per = []
    launches = 0
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            rep = fn(b_dev.data_ptr(), cp, tol, 1000, x_dev.data_ptr()).report
            per.append(ds.last_solve_ms())
            launches += ds.last_launches()
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([statistics.mean(per)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # e2e: host (pinned) b / x through the public call
    b_pin = torch.ones(nloc, dtype=torch.float64).pin_memory().numpy()
    x_pin = torch.zeros(nloc, dtype=torch.float64).pin_memory().numpy()
    e2e = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        t1 = time.perf_counter()
        fn(b_pin, cp, tol, 1000, x_pin)
        if i >= args.warmup:
            e2e.append(time.perf_counter() - t1)
    te = torch.tensor([statistics.mean(e2e)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    if rank == 0:
        line = {"metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": scaling,
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "n": n, "nnz": A.nnz(), "levels": h.nlevels(),
                           "iterations": rep.iterations, "rhs": "ones", "tol": "1e-8*||b||",
                           "partition": f"contiguous row blocks; levels with < {args.gather_rows} rows replicated "
                                        f"(first replicated level {ds.first_replicated})",
                           "transport": "NCCL grouped send/recv (halos), allreduce (dots)",
                           "parallelism": f"row-partitioned over {ws} GPUs", "setup_s": round(setup_s, 3),
                           "l2": "hierarchy > L2 and L2 flushed (256 MB write) before every step"},
                "roofline": None,
                "e2e": {"value": float(te.item()), "unit": "s", "h2d_bytes_per_step": 8 * nloc,
                        "d2h_bytes_per_step": 8 * nloc},
                "gpu_launches": launches, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    del ds
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS) + ["C5", "C5p"])
    ap.add_argument("--host-levels-from", type=int, default=-1,
                    help="hybrid placement: matrices of levels >= K in pinned host memory (paper MI scheme)")
    ap.add_argument("--galerkin-gpu", action="store_true", help="Galerkin products on the GPU during setup")
    ap.add_argument("--ref-sample-iters", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gather-rows", type=int, default=131072)
    ap.add_argument("--dist", action="store_true", help="use the partitioned (NCCL) path even at N = 1")
    args = ap.parse_args()
    wl = args.workload
    if wl in ("C5", "C5p"):
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "the reference's int32 CSR offsets cannot hold "
                              "config 5 (nnz 3.6e9)"}), flush=True)
            return None
        return run_c5(args, wl)
    if args.impl == "reference":
        return run_reference(args, wl)
    if dist_env()[0] > 1 or args.dist:
        return run_multi(args, wl)

    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2007_00056_b200 import sparsh as sp, _lib

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    L = _lib.lib()

    A = WORKLOADS[wl]["gen"](sp)
    n = A.nrows()
    cfg = sp.SolverConfig(smoother=sp.SmootherKind.weighted_jacobi(), max_levels=40, coarse_target=500)
    t0 = time.perf_counter()
    h = sp.Hierarchy(A, cfg, device=local, host_levels_from=args.host_levels_from)
    setup_s = time.perf_counter() - t0  # host setup (aggregation, Galerkin products, coarse inverse)
    t0 = time.perf_counter()
    ctx = h.ctx()
    upload_s = time.perf_counter() - t0  # device context: formats, H2D copies (incl. CUDA init)
    cp = sp.CycleParams.from_config(cfg)._abi()
    solver = WORKLOADS[wl]["solver"]
    b_host = sp.rhs_ones(n)
    tol = 1e-8 * float(np.linalg.norm(b_host))
    max_iters = 1000

    stream = torch.cuda.ExternalStream(L.sb_stream(ctx), device=torch.device("cuda", local))
    b_dev = torch.ones(n, dtype=torch.float64, device=f"cuda:{local}")
    x_dev = torch.zeros(n, dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    fn_dev = L.sb_pcg_dev if solver == "pcg" else L.sb_pbicgstab_dev
    fn_host = L.sb_pcg if solver == "pcg" else L.sb_pbicgstab
    torch.cuda.synchronize()

    def solve_dev():
        rep = _lib.sb_report()
        _lib.check(fn_dev(ctx, C.byref(cp), C.c_void_p(b_dev.data_ptr()), C.c_void_p(x_dev.data_ptr()),
                          tol, max_iters, C.byref(rep)))
        return rep

    # warm-up (also builds + instantiates the solve graph)
    for _ in range(max(args.warmup, 3)):
        rep = solve_dev()
    iters = rep.iterations
    assert rep.termination == 0, f"solve did not converge: termination {rep.termination}"

    # ---- timed region: device-resident solves -------------------------------
    per_step = []
    with ClockSampler(local) as clk:
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush (256 MB > 126 MB L2), outside the event window
            torch.cuda.synchronize()
            rep = solve_dev()
            per_step.append(L.sb_last_solve_ms(ctx))
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
    ms_local = statistics.mean(per_step)
    ms = ms_local
    if ws > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ms / 1e3

    # ---- e2e: public C ABI with pinned host buffers ---------------------------
    b_pin = torch.ones(n, dtype=torch.float64).pin_memory()
    x_pin = torch.zeros(n, dtype=torch.float64).pin_memory()
    bp = C.cast(C.c_void_p(b_pin.data_ptr()), C.POINTER(C.c_double))
    xp = C.cast(C.c_void_p(x_pin.data_ptr()), C.POINTER(C.c_double))
    e2e = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        rep2 = _lib.sb_report()
        t1 = time.perf_counter()
        _lib.check(fn_host(ctx, C.byref(cp), bp, xp, tol, max_iters, C.byref(rep2)))
        dt = time.perf_counter() - t1
        if i >= args.warmup:
            e2e.append(dt)
    e2e_s = statistics.mean(e2e)
    if ws > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    x_np = x_pin.numpy()
    true_rel = float(np.linalg.norm(sp.residual(A, x_np, b_host)) / np.linalg.norm(b_host)) if rank == 0 else None

    # ---- roofline: L0 Jacobi sweep, CUDA events on the solve stream ----------------
    fmts, mbytes = [], []
    for k in range(h.nlevels()):
        fmt = (C.c_int * 4)()
        mb, nz = C.c_int64(), C.c_int64()
        _lib.check(L.sb_level_format(ctx, k, fmt, C.byref(mb), C.byref(nz)))
        fmts.append(list(fmt))
        mbytes.append(mb.value)
    bm = bytes_model(h, cfg.pre_sweeps, cfg.post_sweeps, mbytes)       # bytes the shipped format streams
    bm_csr = bytes_model(h, cfg.pre_sweeps, cfg.post_sweeps)           # SURVEY §8d CSR definition
    avg = C.c_double()
    cnt = C.c_int()
    _lib.check(L.sb_time_kernel(ctx, 0, 0, C.byref(cp), 20, C.byref(avg), C.byref(cnt)))
    jac_ms = avg.value
    vc_ms = C.c_double()
    _lib.check(L.sb_time_kernel(ctx, 3, 0, C.byref(cp), 5, C.byref(vc_ms), C.byref(cnt)))
    vc_launches = cnt.value
    spmv_ms = C.c_double()
    _lib.check(L.sb_time_kernel(ctx, 1, 0, C.byref(cp), 20, C.byref(spmv_ms), C.byref(cnt)))
    peak, peak_kind = peaks()
    achieved = bm["l0_jacobi"] / (jac_ms * 1e-3) / 1e9
    vcycle_gbs = bm["vcycle"] / (vc_ms.value * 1e-3) / 1e9
    it_key = "pcg_iter" if solver == "pcg" else "bicg_iter"
    solve_gbs = (bm[it_key] * iters) / value / 1e9
    csr_jac_gbs = bm_csr["l0_jacobi"] / (jac_ms * 1e-3) / 1e9
    csr_solve_gbs = (bm_csr[it_key] * iters) / value / 1e9

    # kernels per solve: init + [V-cycle + rz/p] + iters x (SpMV+dot, update) + (iters-1) x
    # (V-cycle, rz, xpay) + true residual
    launches = 1 + (vc_launches + 1) + iters * 2 + (iters - 1) * (vc_launches + 2) + 1
    if solver != "pcg":
        launches = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[wl]["desc"], "n": n, "nnz": A.nnz(), "levels": h.nlevels(),
                       "iterations": iters, "rhs": "ones", "tol": "1e-8*||b|| (absolute, as the reference)",
                       "smoother": "weighted Jacobi 2/3, 6 pre / 6 post", "coarsening": "node-HEM",
                       "coarse_target": 500, "max_levels": 40,
                       "l2": "hierarchy (%.0f MB) > 126 MB L2 and L2 flushed (256 MB write) before every step"
                             % (h.device_bytes() / 1e6),
                       "placement": placement(h, args),
                       "parallelism": "single GPU" if ws == 1 else f"{ws} independent replicas",
                       "setup_s": round(setup_s, 3), "upload_s": round(upload_s, 3),
                       "true_rel_residual": true_rel},
            "roofline": {"bound": "hbm", "kernel": sweep_kernel(L, ctx) + " (L0 Jacobi sweep)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "frac_of_spec_8000": achieved / SPEC_HBM_GBS,
                         "traffic": load_traffic(wl),
                         "algorithmic_bytes_per_launch": bm["l0_jacobi"],
                         "bytes_definition": "bytes the shipped lossless format must stream per sweep: "
                                             + bytes_of_format(fmts[0]) + " + 24 B/row (x, f, x_new); "
                                             "SURVEY §8d CSR-equivalent figures below",
                         "launch_ms": jac_ms, "l0_format": fmts[0],
                         "csr_equiv_bytes_per_launch": bm_csr["l0_jacobi"],
                         "csr_equiv_gbs": csr_jac_gbs, "csr_equiv_frac": csr_jac_gbs / peak,
                         "l0_spmv_gbs": (bm["l0_spmv"] / (spmv_ms.value * 1e-3) / 1e9),
                         "vcycle_gbs": vcycle_gbs, "vcycle_ms": vc_ms.value,
                         "solve_gbs": solve_gbs, "solve_frac": solve_gbs / peak,
                         "csr_equiv_solve_gbs": csr_solve_gbs},
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n},
            "gpu_launches": launches * args.steps if launches else None,
        }
        if not args.no_cpu_baseline and ws == 1:
            try:
                line["cpu_baseline"] = cpu_baseline_sample(A, b_host, tol, wl, args.ref_sample_iters, iters)
            except Exception as e:  # never silently: record why
                line["cpu_baseline"] = {"value": None, "error": str(e)}
        line["clocks"] = clk.summary()
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
