"""Rounding sensitivity of the reference's sparse driver (solve(CsrMatrix), RCM +
sparse Cholesky f_T) on the sparse golden cases: the reference's own iteration
counts when every diagonal entry of A is perturbed by +-1 binary32 ulp (7 seeds)
-- the size of the rounding the fp32 factor and the fp32 sandwich already carry.
Writes sensitivity_sparse.json; tests/test_gpu_spchol.py derives its iteration
band from it (max(2, 2 x the largest spread), the policy of DESIGN.md §4.2).

    python tests/golden/make_sparse_sensitivity.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import Oracle, Problem  # noqa: E402
from problems import lap_csr, random_spd_csr  # noqa: E402

CASES = {
    "splap2d50-mplobpcg-schol": (lambda: lap_csr(50, 50), dict(k=10, block=15, tol=1e-12, maxit=500, seed=7)),
    "sprand2000-mplobpcg-schol": (lambda: random_spd_csr(2000, 3, 11), dict(k=8, tol=1e-10, maxit=500, seed=2)),
    "splap3d16-mplobpcg-schol": (lambda: lap_csr(16, 16, 16), dict(k=10, block=16, tol=1e-10, maxit=500)),
}


def main():
    o = Oracle("ref")
    out = {}
    for name, (make, kw) in CASES.items():
        rp, ci, v = make()
        n = rp.size - 1
        d = np.repeat(np.arange(n), np.diff(rp)) == ci
        base = o.solve(Problem.csr(rp, ci, v), "mplobpcg-schol", native=True, **kw)
        runs = []
        for seed in range(1, 8):
            vv = v.copy()
            vv[d] *= 1 + np.random.default_rng(seed).choice([-1, 1], d.sum()) * 2.0 ** -23
            r = o.solve(Problem.csr(rp, ci, vv), "mplobpcg-schol", native=True, **kw)
            runs.append([int(r.iters_lower), int(r.iters_working)])
        ref_total = int(base.iters_lower + base.iters_working)
        out[name] = {"reference": [int(base.iters_lower), int(base.iters_working)],
                     "fp32ulp_runs": runs,
                     "spread": max(abs(a + b - ref_total) for a, b in runs)}
        print(name, out[name], flush=True)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "sensitivity_sparse.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
