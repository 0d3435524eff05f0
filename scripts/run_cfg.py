"""Quick experiment driver: one solve on a named config, prints iterations and time."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2302_12528_b200 as mp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--prob", default="lap2d:1024")
ap.add_argument("--k", type=int, default=32)
ap.add_argument("--block", type=int, default=0)
ap.add_argument("--tol", type=float, default=1e-10)
ap.add_argument("--maxit", type=int, default=20000)
ap.add_argument("--variant", default="mplobpcg-schol")
ap.add_argument("--every", type=int, default=500)
a = ap.parse_args()
kind, dims = a.prob.split(":")
dims = [int(x) for x in dims.split("x")]
A = mp.laplace2d(*dims) if kind == "lap2d" else mp.laplace3d(*dims)
cfg = mp.SolverConfig(k=a.k, block=a.block, tol=a.tol, maxit=a.maxit, variant=a.variant)
t0 = time.time()
r = mp.solve(A, cfg, want_X=False)
t = time.time() - t0
print(f"{a.prob} {a.variant} k={a.k} conv={r.converged} iters={r.iterations_lower}+{r.iterations_working} "
      f"wall={t:.2f}s total={r.timings.total:.2f}s ortho={r.timings.orthogonalize:.2f}s "
      f"eig={r.timings.projected_eig:.2f}s prec={r.timings.precond_apply:.2f}s "
      f"theta0={r.theta[0]:.15e} est={r.a_norm_estimate:.6f}")
h = r.history
for i in range(0, len(h), a.every):
    rn = np.array(h[i].residual_norms[:a.k])
    print(f"  it {i:6d} stage {h[i].stage} n_c {h[i].n_converged:3d} max_res {rn.max():.3e} "
          f"theta_k {h[i].ritz_values[a.k - 1]:.10e}")
