"""A/B of execution options on cfg1 solve time (GPU box helper):
python scripts/ab_options.py key=v1,v2 [reps]"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2302_12528_b200 as mp  # noqa: E402

key, vals = sys.argv[1].split("=")
vals = [int(v) for v in vals.split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = mp.default_context()
A = mp.laplace3d(32)
cfg = mp.SolverConfig(k=10, block=16, tol=1e-10, maxit=2000, variant="mplobpcg-schol")
res = {v: [] for v in vals}
for r in range(reps + 1):
    for v in vals:
        ctx.set_option(key, v)
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = mp.solve(A, cfg, want_X=False, history=False)
        torch.cuda.synchronize()
        if r:
            res[v].append((time.perf_counter() - t, out.iterations_lower + out.iterations_working))
for v in vals:
    ts = sorted(x[0] for x in res[v])
    it = res[v][0][1]
    print(f"{key}={v}: median {1e3 * ts[len(ts) // 2]:.1f} ms  iterations {it}  per-iteration {1e6 * ts[len(ts) // 2] / it:.1f} us")
