"""Compare the GPU's per-iteration history with the reference golden history
(GPU box helper): python scripts/cmp_hist.py lap3d16-mplobpcg-schol [every]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2302_12528_b200 as mp  # noqa: E402
from conftest import load_golden  # noqa: E402
from test_gpu_solver import make_op  # noqa: E402

name = sys.argv[1]
every = int(sys.argv[2]) if len(sys.argv) > 2 else 10
g = load_golden(name)
kw = eval(str(g["kw"]))
cfg = mp.SolverConfig(variant=str(g["variant"]), **kw)
r = mp.solve(make_op(mp, name), cfg)
gs, gnc, gres, gritz = g["hist_stage"], g["hist_nc"], g["hist_resid"], g["hist_ritz"]
hs = [h.stage for h in r.history]
hnc = [h.n_converged for h in r.history]
hres = np.array([h.residual_norms for h in r.history])
hritz = np.array([h.ritz_values for h in r.history])
k = cfg.k
print(f"{name}: ref {int(g['iters_lower'])}+{int(g['iters_working'])}  gpu {r.iterations_lower}+{r.iterations_working}")
print(" it | ref st nc  max_res(k)   theta_k-1     | gpu st nc  max_res(k)   theta_k-1")
n = max(len(gs), len(hs))
for i in range(0, n, every):
    a = (f"{gs[i]:2d} {gnc[i]:2d} {gres[i][:k].max():.3e} {gritz[i][k - 1]:.10f}" if i < len(gs) else " " * 38)
    b = (f"{hs[i]:2d} {hnc[i]:2d} {hres[i][:k].max():.3e} {hritz[i][k - 1]:.10f}" if i < len(hs) else "")
    print(f"{i:4d} | {a} | {b}")
