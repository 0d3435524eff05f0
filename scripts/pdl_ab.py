"""cfg1 time-to-solution with and without programmatic edges in the iteration
graphs (process option "pdl"), same process, alternating; results must agree bitwise."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp  # noqa: E402

ctx = mp.default_context()
A = mp.laplace3d(32)
cfg = mp.SolverConfig(k=10, block=16, tol=1e-10, maxit=2000, variant="mplobpcg-schol")
T = mp.jacobi(A, mp.LOWER)
res = {0: [], 1: [], 2: []}
th = {}
import os
KEY = os.environ.get("AB_KEY", "pdl").encode()
VALS = [int(v) for v in os.environ.get("AB_VALS", "0,1,2").split(",")]
res = {v: [] for v in VALS}
for rep in range(4):
    for opt in VALS:
        assert ctx.lib.mpeig_set_process_option(KEY, opt) == 0
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = mp.solve(A, cfg, T=T, want_X=False, history=False)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        if rep:
            res[opt].append(dt)
        th.setdefault(opt, (r.iterations_lower, r.iterations_working, r.theta.copy()))
for opt in VALS:
    print(f"{KEY.decode()}={opt}: median {np.median(res[opt]):.4f} s  runs {[round(x, 4) for x in res[opt]]}  "
          f"iters {th[opt][:2]}")
print("bitwise equal theta:", all(np.array_equal(th[VALS[0]][2], th[v][2]) for v in VALS))
