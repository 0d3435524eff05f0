import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2302_12528_b200 as mp
for opts in ({"spec_mode": 1}, {"spec_mode": 0}, {"spec_mode": 0, "eig_backend": 1}):
    ctx = mp.Context(0)
    for k, v in opts.items(): ctx.set_option(k, v)
    A = mp.laplace3d(12, ctx=ctx)
    cfg = mp.SolverConfig(k=6, tol=1e-10, maxit=1000, variant="mplobpcg-schol")
    hist = []
    import paper_2302_12528_b200.api as api
    try:
        r = mp.solve(A, cfg)
        print(opts, "OK", r.iterations_lower, r.iterations_working, flush=True)
    except Exception as e:
        print(opts, "ERR", e, flush=True)
    # stage-1 only run
    T = mp.jacobi(A, mp.LOWER)
    X0 = mp.to_device(np.linalg.qr(np.random.default_rng(0).standard_normal((A.n, 9)))[0], dtype=__import__('torch').float32)
    h = []
    st = mp.lobpcg_stage(A, A.n, X0, cfg, T, 6.0, mp.StageOptions(tol=5e-6, stagnation_exit=True, tag=1), history=h)
    Xh = mp.to_host(st.X)
    print("  stage1", st.iterations, st.converged, "nan", np.isnan(Xh).sum(), "colnorms", np.linalg.norm(Xh, axis=0).round(4), flush=True)
    print("  last hist", h[-1].ritz_values[:3], h[-1].residual_norms[:3], h[-1].n_converged, flush=True)
