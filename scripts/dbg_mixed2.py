import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2302_12528_b200 as mp
ctx = mp.Context(0)
ctx.set_option("spec_mode", 0)
A = mp.laplace3d(12, ctx=ctx)
cfg = mp.SolverConfig(k=6, tol=1e-10, maxit=40, variant="mplobpcg-schol")
T = mp.jacobi(A, mp.LOWER)
for m in (9, 10):
    X0 = mp.to_device(np.linalg.qr(np.random.default_rng(0).standard_normal((A.n, m)))[0], dtype=torch.float32)
    h = []
    try:
        st = mp.lobpcg_stage(A, A.n, X0, cfg, T, 6.0, mp.StageOptions(tol=5e-6, stagnation_exit=True, tag=1), history=h)
    except Exception as e:
        print("ERR", e)
    for i, r in enumerate(h[:6]):
        print(m, i, np.round(r.ritz_values[:4], 5), np.array(r.residual_norms[:3]))
