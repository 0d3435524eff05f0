import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import paper_2302_12528_b200 as mp
from conftest import load_golden
g = load_golden("lap3d16-dlobpcg-dchol")
H = {}
for backend in (0, 1):
    ctx = mp.Context(0); ctx.set_option("spec_mode", 0); ctx.set_option("eig_backend", backend)
    A = mp.laplace3d(16, ctx=ctx)
    r = mp.solve(A, mp.SolverConfig(variant="dlobpcg-dchol", k=10, block=16, tol=1e-10, maxit=2000))
    H[backend] = r.history
ref_res = g["hist_resid"]; ref_nc = g["hist_nc"]
for it in range(0, 340, 20):
    row = [f"{it:4d}"]
    for b in (0, 1):
        h = H[b][min(it, len(H[b]) - 1)]
        rn = np.array(h.residual_norms)
        row.append(f"{'jac' if b == 0 else 'cus'} nc {h.n_converged:2d} r0-9 max {rn[:10].max():.2e} r10-15 max {rn[10:].max():.2e}")
    i = min(it, len(ref_nc) - 1)
    row.append(f"ref nc {ref_nc[i]:2d} max {ref_res[i][:10].max():.2e} {ref_res[i][10:].max():.2e}")
    print(" | ".join(row))
