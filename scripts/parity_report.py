"""Print GPU-vs-reference parity for every golden case (diagnostic)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2302_12528_b200 as mp  # noqa: E402
from conftest import load_golden  # noqa: E402
from test_gpu_solver import make_op  # noqa: E402

names = sys.argv[1:] or [f[:-4] for f in sorted(os.listdir(os.path.join(ROOT, "tests", "golden")))
                         if f.endswith(".npz") and f != "pcg64.npz"]
for name in names:
    g = load_golden(name)
    kw = eval(str(g["kw"]))
    cfg = mp.SolverConfig(variant=str(g["variant"]), **kw)
    r = mp.solve(make_op(mp, name), cfg)
    rel = np.abs(r.theta - g["theta"]) / np.abs(g["theta"])
    thr = cfg.tol * (r.a_norm_estimate + np.abs(r.theta))
    hr = np.array([h.ritz_values for h in r.history])
    gr = g["hist_ritz"]
    n = min(len(hr), len(gr))
    div = np.abs(hr[:n] - gr[:n]).max(axis=1) / np.abs(gr[:n]).max()
    first = int(np.argmax(div > 1e-12)) if (div > 1e-12).any() else -1
    print(f"{name:28s} gpu {r.iterations_lower:5d}+{r.iterations_working:5d} ref "
          f"{int(g['iters_lower']):5d}+{int(g['iters_working']):5d} conv {r.converged}/{bool(g['converged'])} "
          f"theta_rel {rel.max():.1e} resid/thr {np.max(r.residual_norms / thr):.3f} "
          f"est_rel {abs(r.a_norm_estimate / float(g['a_norm_est']) - 1):.1e} "
          f"first_div>1e-12@{first} div@10 {div[min(10, n - 1)]:.1e} t={r.timings.total:.2f}s", flush=True)
