import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2302_12528_b200 as mp
from problems import spd_dense
names = ["QL", "jac+tri", "jac+refl", "jac"]
for N, k, m, variant in ((16, 10, 16, "dlobpcg-dchol"), (32, 10, 16, "dlobpcg-dchol"), (16, 10, 16, "mplobpcg-schol"), (32, 10, 16, "mplobpcg-schol"), (8, 4, 6, "dlobpcg-dchol"), (0, 8, 12, "dlobpcg-dchol")):
    row = []
    for meth in range(4):
        ctx = mp.Context(0); ctx.set_option("syev_method", meth)
        A = mp.laplace3d(N, ctx=ctx) if N else mp.dense_matrix(spd_dense(256, 1e3, 5)[0], ctx=ctx)
        cfg = mp.SolverConfig(variant=variant, k=k, block=m, tol=1e-10, maxit=3000, seed=0 if N else 3)
        try:
            r = mp.solve(A, cfg)
            row.append(f"{names[meth]} {r.iterations_lower}+{r.iterations_working} ({r.timings.total:.2f}s)")
        except Exception as e:
            row.append(f"{names[meth]} ERR {e}")
    print(N, variant, " | ".join(row), flush=True)
