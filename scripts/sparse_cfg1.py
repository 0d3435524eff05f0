"""cfg1's matrix (3-D 7-pt Laplacian 32^3, k = 10, m = 16, tol 1e-10) through the
reference's stock SPARSE driver solve(CsrMatrix, cfg) (drivers.hpp:183-210):
RCM-permuted system and the sparse Cholesky preconditioner --
the paper's own preconditioner -- on one B200, next to the reference on one host
core (oracle/_ref, when present).

    python scripts/sparse_cfg1.py [nx] [--ref]
Prints one JSON line per variant: factor + solve time (wall clock around the
synchronous call), iterations, theta vs the reference, per-kernel-class shares.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_12528_b200 as mp  # noqa: E402
from problems import lap_csr  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    nx = int(args[0]) if args else 32
    rp, ci, v = lap_csr(nx, nx, nx)
    for variant in ("mplobpcg-schol", "dlobpcg-dchol"):
        cfg = mp.SolverConfig(variant=variant, k=10, block=16, tol=1e-10, maxit=500, seed=0)
        mp.solve_csr(rp, ci, v, cfg, want_X=False)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = mp.solve_csr(rp, ci, v, cfg, want_X=False)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        with mp.profile():
            mp.solve_csr(rp, ci, v, cfg, want_X=False)
        rep = mp.profile.report()
        tot = sum(x["ms"] for x in rep.values()) or 1.0
        kern = {k: {"launches": x["count"], "share": round(x["ms"] / tot, 4),
                    "ms_per_launch": round(x["ms"] / max(x["count"], 1), 4)}
                for k, x in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])}
        out = {"workload": f"3-D 7-pt Laplacian {nx}^3 CSR, k=10, m=16, tol 1e-10, "
                           f"solve(CsrMatrix): RCM + sparse Cholesky f_T",
               "variant": variant, "converged": r.converged,
               "iterations": {"lower": r.iterations_lower, "working": r.iterations_working},
               "solve_incl_factor_s": round(t, 4), "theta0": float(r.theta[0]),
               "kernels_ms_total": round(tot, 2), "kernels": kern}
        if "--ref" in sys.argv:
            from oracle import Oracle, Problem, available
            if available("ref"):
                t0 = time.perf_counter()
                g = Oracle("ref").solve(Problem.csr(rp, ci, v), variant, k=10, block=16,
                                        tol=1e-10, maxit=500, seed=0, native=True)
                out["reference"] = {
                    "seconds_1_core": round(time.perf_counter() - t0, 3),
                    "factor_s": round(g.t_setup, 3),
                    "iterations": {"lower": int(g.iters_lower), "working": int(g.iters_working)},
                    "theta_max_rel_diff": float(np.max(np.abs(r.theta - g.theta) / np.abs(g.theta)))}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
