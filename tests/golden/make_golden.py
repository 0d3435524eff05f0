"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libmpeig_ref.so, built from
/root/reference/proj by oracle/Makefile) through its own lobpcg_stage /
BlockOperator API (oracle/ref_harness.cpp) and stores the results as small
.npz files.  The GPU box has no /root/reference; the fixtures travel instead.

    python tests/golden/make_golden.py            # fast set (< 1 min)
    python tests/golden/make_golden.py --case cfg1-dlobpcg-dchol   # one long case

Each fixture holds: theta, resid, iteration counts, converged, a_norm_est,
the full per-iteration history (stage, n_c, dropped, rotation fallback, Ritz
values, residual norms) and the reference's own wall time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle, Problem  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests"))
from problems import lap_csr, random_spd_csr, spd_dense  # noqa: E402
from paper_2302_12528_b200.generators import ks_csr  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


CASES = {
    # name: (problem factory, variant, solve kwargs)
    "lap3d8-dlobpcg-dchol": (lambda: Problem.lap3d(8), "dlobpcg-dchol", dict(k=4, tol=1e-10, maxit=500)),
    "lap3d8-dlobpcg-schol": (lambda: Problem.lap3d(8), "dlobpcg-schol", dict(k=4, tol=1e-10, maxit=500)),
    "lap3d8-mplobpcg-schol": (lambda: Problem.lap3d(8), "mplobpcg-schol", dict(k=4, tol=1e-10, maxit=500)),
    "lap3d8-pinvit": (lambda: Problem.lap3d(8), "pinvit", dict(k=4, tol=1e-10, maxit=5000)),
    "lap3d16-dlobpcg-dchol": (lambda: Problem.lap3d(16), "dlobpcg-dchol", dict(k=10, block=16, tol=1e-10, maxit=2000)),
    "lap3d16-dlobpcg-schol": (lambda: Problem.lap3d(16), "dlobpcg-schol", dict(k=10, block=16, tol=1e-10, maxit=2000)),
    "lap3d16-mplobpcg-schol": (lambda: Problem.lap3d(16), "mplobpcg-schol", dict(k=10, block=16, tol=1e-10, maxit=2000)),
    "lap2d50-mplobpcg-schol": (lambda: Problem.lap2d(50), "mplobpcg-schol", dict(k=10, block=15, tol=1e-12, maxit=600, seed=7)),
    "lap2d50-dlobpcg-dchol": (lambda: Problem.lap2d(50), "dlobpcg-dchol", dict(k=10, block=15, tol=1e-12, maxit=600, seed=7)),
    "lap2d5x500-mplobpcg-schol": (lambda: Problem.lap2d(5, 500), "mplobpcg-schol", dict(k=5, block=8, tol=1e-10, maxit=8000, seed=1)),
    "dense256-dlobpcg-dchol": (lambda: Problem.dense_matrix(spd_dense(256, 1e3, 5)[0]), "dlobpcg-dchol", dict(k=8, tol=1e-10, maxit=2000, seed=3)),
    "dense256-mplobpcg-schol": (lambda: Problem.dense_matrix(spd_dense(256, 1e3, 5)[0]), "mplobpcg-schol", dict(k=8, tol=1e-10, maxit=2000, seed=3)),
    "lap2d32-pinvit": (lambda: Problem.lap2d(32), "pinvit", dict(k=4, block=6, tol=1e-8, maxit=400)),
    # the reference's own dense Cholesky preconditioner (stock solve(DenseMatrix),
    # drivers.hpp:158-181): fp64 factor (dchol), fp32 factor (schol,
    # mixed, PINVIT), and an ill-conditioned case whose fp32 factor needs
    # retry_dense's shift (precond.hpp:140-146)
    "dense256chol-dlobpcg-dchol": (lambda: Problem.dense_matrix(spd_dense(256, 1e3, 5)[0]), "dlobpcg-dchol", dict(k=8, tol=1e-10, maxit=500, seed=3, native=True)),
    "dense256chol-dlobpcg-schol": (lambda: Problem.dense_matrix(spd_dense(256, 1e3, 5)[0]), "dlobpcg-schol", dict(k=8, tol=1e-10, maxit=500, seed=3, native=True)),
    "dense256chol-mplobpcg-schol": (lambda: Problem.dense_matrix(spd_dense(256, 1e3, 5)[0]), "mplobpcg-schol", dict(k=8, tol=1e-10, maxit=500, seed=3, native=True)),
    "dense256chol-pinvit": (lambda: Problem.dense_matrix(spd_dense(256, 1e3, 5)[0]), "pinvit", dict(k=8, tol=1e-10, maxit=500, seed=3, native=True)),
    "dense256chol-k1e10-dlobpcg-schol": (lambda: Problem.dense_matrix(spd_dense(256, 1e10, 5)[0]), "dlobpcg-schol", dict(k=8, tol=1e-10, maxit=12, seed=3, native=True)),
    # the reference's stock sparse driver solve(CsrMatrix) (drivers.hpp:183-210): RCM
    # permutation + its own sparse Cholesky preconditioner; the last
    # case is shifted to lambda_min = -1e-6, so the fp32 factor needs retry_sparse's shift
    "splap3d16-dlobpcg-dchol": (lambda: Problem.csr(*lap_csr(16, 16, 16)), "dlobpcg-dchol", dict(k=10, block=16, tol=1e-10, maxit=500, native=True)),
    "splap3d16-dlobpcg-schol": (lambda: Problem.csr(*lap_csr(16, 16, 16)), "dlobpcg-schol", dict(k=10, block=16, tol=1e-10, maxit=500, native=True)),
    "splap3d16-mplobpcg-schol": (lambda: Problem.csr(*lap_csr(16, 16, 16)), "mplobpcg-schol", dict(k=10, block=16, tol=1e-10, maxit=500, native=True)),
    "splap3d16-pinvit": (lambda: Problem.csr(*lap_csr(16, 16, 16)), "pinvit", dict(k=10, block=16, tol=1e-10, maxit=500, native=True)),
    "splap2d50-mplobpcg-schol": (lambda: Problem.csr(*lap_csr(50, 50)), "mplobpcg-schol", dict(k=10, block=15, tol=1e-12, maxit=500, seed=7, native=True)),
    "sprand2000-mplobpcg-schol": (lambda: Problem.csr(*random_spd_csr(2000, 3, 11)), "mplobpcg-schol", dict(k=8, tol=1e-10, maxit=500, seed=2, native=True)),
    "splap3d8indef-dlobpcg-schol": (lambda: Problem.csr(*lap_csr(8, 8, 8, shift=0.3618452752845494)), "dlobpcg-schol", dict(k=4, tol=1e-10, maxit=6, native=True)),
    # north-star block sizes (SURVEY §8d ladder): m = 48 (cfg2 family, 3m = 144 > 96:
    # the large-block path) and m = 96 with the reference's dense Cholesky (cfg3 family)
    "lap2d64k32-dlobpcg-dchol": (lambda: Problem.lap2d(64), "dlobpcg-dchol", dict(k=32, block=48, tol=1e-10, maxit=5000)),
    "lap2d64k32-mplobpcg-schol": (lambda: Problem.lap2d(64), "mplobpcg-schol", dict(k=32, block=48, tol=1e-10, maxit=5000)),
    "lap2d64k32-pinvit": (lambda: Problem.lap2d(64), "pinvit", dict(k=32, block=48, tol=1e-10, maxit=150)),
    "lap2d128k32-dlobpcg-dchol": (lambda: Problem.lap2d(128), "dlobpcg-dchol", dict(k=32, block=48, tol=1e-10, maxit=8000)),
    "dense2048chol-dlobpcg-dchol": (lambda: Problem.dense_matrix(spd_dense(2048, 1e3, 9)[0]), "dlobpcg-dchol", dict(k=64, tol=1e-10, maxit=500, seed=5, native=True)),
    "dense2048chol-mplobpcg-schol": (lambda: Problem.dense_matrix(spd_dense(2048, 1e3, 9)[0]), "mplobpcg-schol", dict(k=64, tol=1e-10, maxit=500, seed=5, native=True)),
    # cfg5 family (BASELINE.json configs[4]): the Kohn-Sham-like H = -Laplacian + V
    # (paper_2302_12528_b200/generators.py), clustered low spectrum, 32^3, k = 16
    "ks32-dlobpcg-dchol": (lambda: Problem.csr(*ks_csr(32, 32, 32, seed=0)), "dlobpcg-dchol", dict(k=16, block=24, tol=1e-10, maxit=4000)),
    "ks32-mplobpcg-schol": (lambda: Problem.csr(*ks_csr(32, 32, 32, seed=0)), "mplobpcg-schol", dict(k=16, block=24, tol=1e-10, maxit=4000)),
    # cfg 1 (BASELINE.json configs[0]) -- minutes each on one core
    "cfg1-dlobpcg-dchol": (lambda: Problem.lap3d(32), "dlobpcg-dchol", dict(k=10, block=16, tol=1e-10, maxit=2000)),
    "cfg1-dlobpcg-schol": (lambda: Problem.lap3d(32), "dlobpcg-schol", dict(k=10, block=16, tol=1e-10, maxit=2000)),
    "cfg1-mplobpcg-schol": (lambda: Problem.lap3d(32), "mplobpcg-schol", dict(k=10, block=16, tol=1e-10, maxit=2000)),
}
LARGE = ["ks32-dlobpcg-dchol", "ks32-mplobpcg-schol", "lap2d64k32-dlobpcg-dchol", "lap2d64k32-mplobpcg-schol", "lap2d64k32-pinvit",
         "lap2d128k32-dlobpcg-dchol", "dense2048chol-dlobpcg-dchol", "dense2048chol-mplobpcg-schol"]
FAST = [c for c in CASES if not c.startswith("cfg1") and c not in LARGE]


def run(name: str) -> None:
    make, variant, kw = CASES[name]
    prob = make()
    r = Oracle("ref").solve(prob, variant, **kw)
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"),
        variant=variant, kw=repr(kw), status=r.status, msg=r.msg, converged=r.converged,
        iters_lower=r.iters_lower, iters_working=r.iters_working, a_norm_est=r.a_norm_est,
        theta=r.theta, resid=r.resid, hist_stage=r.hist_stage, hist_nc=r.hist_nc,
        hist_dropped=r.hist_dropped, hist_fallback=r.hist_fallback,
        hist_ritz=r.hist_ritz, hist_resid=r.hist_resid, t_total=r.t_total,
        precond_shift=r.extra["t_stage1"] if kw.get("native") else 0.0)
    print(f"{name}: status={r.status} conv={r.converged} iters={r.iters_lower}+{r.iters_working} "
          f"theta0={r.theta[0]!r} t={r.t_total:.2f}s", flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append")
    ap.add_argument("--rcm", action="store_true", help="also write rcm.npz with --case")
    a = ap.parse_args()
    for name in a.case or FAST:
        run(name)
    # PCG64 golden outputs (tests/test_precision.cpp:56-71 values are asserted
    # in tests/test_oracle.py; these are the longer streams)
    o = Oracle("ref")
    if a.rcm or not a.case:
        rcm = {}
        for nm, (rp, ci, _) in (("lap3d8", lap_csr(8, 8, 8)), ("lap2d5x500", lap_csr(5, 500)),
                                ("lap3d12x7x5", lap_csr(12, 7, 5)),
                                ("rand2000", random_spd_csr(2000, 3, 11))):
            perm = np.zeros(rp.size - 1, np.int64)
            o.fn("rcm")(C.c_int64(rp.size - 1), rp.ctypes.data_as(C.c_void_p),
                        ci.ctypes.data_as(C.c_void_p), perm.ctypes.data_as(C.c_void_p))
            rcm[nm] = perm
        np.savez_compressed(os.path.join(OUT, "rcm.npz"), **rcm)
    if a.case:
        return
    np.savez_compressed(os.path.join(OUT, "pcg64.npz"),
                        s0=o.pcg64(0, 64), s42=o.pcg64(42, 64), s2026=o.pcg64(2026, 64),
                        gauss_0_33x5=o.gaussian(33, 5, 0),
                        gauss_sketch=o.gaussian(40, 8, 0 ^ 0x9E3779B97F4A7C15))


if __name__ == "__main__":
    main()
