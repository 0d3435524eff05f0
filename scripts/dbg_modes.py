import sys, traceback
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2302_12528_b200 as mp
for variant in ["dlobpcg-dchol", "mplobpcg-schol"]:
    for opts in ({"spec_mode": 1, "use_graphs": 1}, {"spec_mode": 1, "use_graphs": 0}, {"spec_mode": 0, "use_graphs": 0}):
        try:
            ctx = mp.Context(0)
            for k, v in opts.items(): ctx.set_option(k, v)
            A = mp.laplace3d(12, 11, 10, ctx=ctx)
            r = mp.solve(A, mp.SolverConfig(k=6, tol=1e-10, maxit=800, variant=variant))
            print(variant, opts, r.converged, r.iterations_lower, r.iterations_working, r.theta[:3], flush=True)
        except Exception as e:
            print(variant, opts, "ERR", type(e).__name__, e, flush=True)
