"""One cfg1 solve (after one warm-up) -- the command profiled by ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2302_12528_b200 as mp  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "mplobpcg-schol"
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
A = mp.laplace3d(32)
cfg = mp.SolverConfig(k=10, block=16, tol=1e-10, maxit=maxit, variant=variant)
for _ in range(2):
    r = mp.solve(A, cfg, want_X=False, history=False)
print(variant, r.converged, r.iterations_lower, r.iterations_working, r.theta[0])
