import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
os.environ["MPEIG_DEBUG_SPEC"] = "1"
import paper_2302_12528_b200 as mp
for graphs in (0, 1):
    ctx = mp.Context(0); ctx.set_option("syev_method", 0); ctx.set_option("use_graphs", graphs)
    A = mp.laplace3d(16, ctx=ctx)
    try:
        r = mp.solve(A, mp.SolverConfig(variant="dlobpcg-dchol", k=10, block=16, tol=1e-10, maxit=3000))
        print("graphs", graphs, "ok", r.iterations_working, flush=True)
    except Exception as e:
        print("graphs", graphs, "ERR", e, flush=True)
