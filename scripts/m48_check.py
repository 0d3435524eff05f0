import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2302_12528_b200 as mp
ctx = mp.default_context()
for opt in (10, 0):
    ctx.set_option("spec_qr", opt)
    for variant in ("mplobpcg-schol", "dlobpcg-dchol"):
        A = mp.laplace3d(40)
        cfg = mp.SolverConfig(k=32, block=48, tol=1e-10, maxit=20000, variant=variant)
        ctx.spec_rollbacks(reset=True)
        t = time.time()
        r = mp.solve(A, cfg, want_X=False)
        print(f"spec_qr={opt} {variant}: conv={r.converged} iters={r.iterations_lower}+{r.iterations_working} "
              f"theta0={r.theta[0]:.15e} theta31={r.theta[31]:.15e} rollbacks={ctx.spec_rollbacks()} {time.time()-t:.1f}s", flush=True)
