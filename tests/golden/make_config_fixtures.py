"""TEST INFRASTRUCTURE: golden fixtures of the REFERENCE at the BASELINE configs.

Runs the reference's own code (oracle/_ref/libsparsh_ref.so = the unmodified
sparsh headers, -O3 -ffp-contract=off) once per configuration and records what
the GPU parity tests (tests/test_gpu_configs.py) assert against:

* setup: per level n, nnz and CRC32 of row_ptr / col_idx / values / fine_to_coarse
  (aggregates and coarse operators must be bit-exact);
* the solve to 1e-8 * ||b|| (rhs ones, x0 = 0; PCG, or PBiCGStab for C4):
  iterations, termination, residual history, true residual, wall time and
  thread count (inc/krylov.hpp:65-119 / 126-211);
* the solution x_k at the reference's final iteration: a strided sample
  (every `stride`-th entry), ||x||_2, sum(x) and x . g for the seeded
  g = default_rng(20070056).standard_normal(n); the same for the
  equal-iteration run (tol = 1e-300, max_iters = k_ref: "xe"), which differs
  from the to-tolerance iterate only for a BiCGStab half-step exit.

The matrices come from oracle/ref_capi.cpp (triplets through the reference's
CsrMatrix::from_triplets), so the product library is not involved.

  python tests/golden/make_config_fixtures.py [C1 C2 C3 C4 T256 P27_128]

Runtimes on the 8-core build container: C1/C2 ~25 s, P27_128 ~1 min,
T256 ~4 min, C3 ~5 min, C4 ~6 min.
"""
import json
import os
import sys
import time
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

SOLVER = {"C1": "pcg", "C2": "pcg", "C3": "pcg", "C4": "pbicgstab", "T256": "pcg", "P27_128": "pcg"}
SAMPLES = 16384


def crc(a):
    return int(zlib.crc32(np.ascontiguousarray(a).view(np.uint8)))


def g_vector(n):
    return np.random.default_rng(20070056).standard_normal(n)


def main(names):
    import oracle as orc
    R = orc.Ref()
    threads = os.cpu_count() or 1
    R.set_threads(threads)
    for name in names:
        t0 = time.perf_counter()
        A = R.problem(name)
        n, nnz = A.nrows(), A.nnz()
        t_gen = time.perf_counter() - t0
        t0 = time.perf_counter()
        h = R.hierarchy(A, 500, 40)
        t_setup = time.perf_counter() - t0
        levels = []
        for k in range(h.nlevels()):
            rp, ci, v, agg = h.level(k)
            levels.append({"n": int(rp.size - 1), "nnz": int(ci.size), "crc_rp": crc(rp), "crc_ci": crc(ci),
                           "crc_v": crc(v), "crc_agg": crc(agg) if agg is not None else None})
        del A
        b = np.ones(n)
        tol = 1e-8 * float(np.linalg.norm(b))
        out = getattr(h, SOLVER[name])(b, tol, 1000)
        x = out.x
        stride = max(1, n // SAMPLES)
        # the equal-iteration solution (tol = 1e-300, max_iters = k_ref; SURVEY §8c
        # protocol). For PCG it is the to-tolerance iterate; BiCGStab's half-step
        # exit (krylov.hpp:167-173) returns x + alpha p~ where the equal-iteration
        # run completes the step, so it is recorded separately.
        xe = x if SOLVER[name] == "pcg" else getattr(h, SOLVER[name])(b, 1e-300, out.iterations).x
        meta = {"name": name, "solver": SOLVER[name], "n": n, "nnz": nnz, "levels": levels,
                "tol": tol, "rhs": "ones", "iterations": out.iterations, "termination": out.termination,
                "true_residual": out.true_residual, "wall_time": out.wall_time, "threads": threads,
                "gen_s": t_gen, "setup_s": t_setup, "stride": stride,
                "x_norm2": float(np.linalg.norm(x)), "x_sum": float(np.sum(x)), "x_dot_g": float(x @ g_vector(n)),
                "xe_norm2": float(np.linalg.norm(xe)), "xe_sum": float(np.sum(xe)), "xe_dot_g": float(xe @ g_vector(n)),
                "generator": "oracle/ref_capi.cpp ref_stencil7/ref_convdiff3d/ref_stencil27/convdiff2d"}
        np.savez_compressed(os.path.join(HERE, f"config_{name}.npz"), x_sample=x[::stride], xe_sample=xe[::stride],
                            residual_history=np.asarray(out.residual_history),
                            time_history=np.asarray(out.time_history), meta=json.dumps(meta))
        print(f"{name}: n={n} levels={len(levels)} {SOLVER[name]} it={out.iterations} term={out.termination} "
              f"wall={out.wall_time:.1f}s setup={t_setup:.1f}s gen={t_gen:.1f}s", flush=True)
        del h, out, x


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "P27_128", "T256", "C3", "C4"])
