"""Rounding-noise floor of the parity contract at the BASELINE configurations.

The reference sums dot products sequentially (inc/csr.hpp:245-251); the GPU
sums them as deterministic trees. This runs the plain-C restatement of the
reference (oracle/sparsh_oracle.c, bit-identical to the reference: mode 0)
and the same restatement with only the dot-product summation order changed
(mode 1: blocks of 256, then a pairwise tree) at the reference's iteration
count (tol = 1e-300, max_iters = k_ref), and reports the relative L2 distance
of the two solutions: how far a legal reordering of the reference's OWN dots
moves x. Writes tests/golden/noise_floor_<name>.json.

  python tools/noise_floor.py C4 [C3 T256 ...]     (single-threaded, minutes each)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as orc  # noqa: E402


def main(names):
    R = orc.Ref()
    for name in names:
        z = np.load(os.path.join(ROOT, "tests", "golden", f"config_{name}.npz"))
        meta = json.loads(str(z["meta"]))
        rp, ci, v = R.problem(name).arrays()
        A = orc.ArraysCsr(rp, ci, v)
        P = orc.Port()
        t0 = time.perf_counter()
        h = P.hierarchy(A, 500, 40)
        b = np.ones(A.nrows())
        k = meta["iterations"]
        out = {}
        for mode in (0, 1):
            P.set_dot_mode(mode)
            out[mode] = getattr(h, meta["solver"])(b, 1e-300, k)
        P.set_dot_mode(0)
        x0, x1 = out[0].x, out[1].x
        rel = float(np.linalg.norm(x0 - x1) / np.linalg.norm(x0))
        ref_x = z["xe_sample"] if "xe_sample" in z.files else z["x_sample"]  # the equal-iteration iterate
        samp = float(np.linalg.norm(x0[::meta["stride"]] - ref_x) / np.linalg.norm(ref_x))
        res = {"name": name, "solver": meta["solver"], "iterations": k, "rel_l2_reordered_dots": rel,
               "port_vs_reference_sample_rel": samp, "seconds": round(time.perf_counter() - t0, 1)}
        with open(os.path.join(ROOT, "tests", "golden", f"noise_floor_{name}.json"), "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C4"])
