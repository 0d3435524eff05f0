import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2302_12528_b200 as mp
for backend in (0, 1):
    ctx = mp.Context(0)
    ctx.set_option("spec_mode", 0)
    ctx.set_option("eig_backend", backend)
    A = mp.laplace3d(12, ctx=ctx)
    cfg = mp.SolverConfig(k=6, tol=1e-10, maxit=300, variant="mplobpcg-schol")
    T = mp.jacobi(A, mp.LOWER)
    X0 = mp.to_device(np.linalg.qr(np.random.default_rng(0).standard_normal((A.n, 9)))[0], dtype=torch.float32)
    h = []
    st = mp.lobpcg_stage(A, A.n, X0, cfg, T, 6.0, mp.StageOptions(tol=5e-6, stagnation_exit=True, tag=1), history=h)
    bad = [i for i, r in enumerate(h) if not np.all(np.isfinite(r.ritz_values))]
    f = bad[0] if bad else len(h)
    print("backend", backend, "iters", st.iterations, "first nan", f)
    for i in range(max(0, f - 4), min(len(h), f + 1)):
        r = h[i]
        print("  ", i, np.array(r.ritz_values), np.array(r.residual_norms[:9]).round(8), r.w_columns_dropped, r.basis_rotation_fallback)
