"""Iteration split of the sparse-Cholesky random-matrix golden case on the device."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2302_12528_b200 as mp  # noqa: E402
from problems import random_spd_csr  # noqa: E402

rp, ci, v = random_spd_csr(2000, 3, 11)
cfg = mp.SolverConfig(variant="mplobpcg-schol", k=8, tol=1e-10, maxit=500, seed=2)
r = mp.solve_csr(rp, ci, v, cfg)
print("sprand2000 mixed", r.iterations_lower, r.iterations_working, "(reference 57 + 64)")
