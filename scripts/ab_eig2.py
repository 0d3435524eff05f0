import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2302_12528_b200 as mp
for N, k, m, variant in ((16, 10, 16, "dlobpcg-dchol"), (32, 10, 16, "dlobpcg-dchol"), (16, 10, 16, "mplobpcg-schol")):
    row = []
    for backend in (0, 1, 2):
        ctx = mp.Context(0); ctx.set_option("spec_mode", 0); ctx.set_option("eig_backend", backend)
        A = mp.laplace3d(N, ctx=ctx)
        r = mp.solve(A, mp.SolverConfig(variant=variant, k=k, block=m, tol=1e-10, maxit=3000))
        row.append(f"{['jacobi','syevd','syevj'][backend]} {r.iterations_lower}+{r.iterations_working}")
    print(N, variant, " | ".join(row), flush=True)
