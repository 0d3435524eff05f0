"""A/B: one-CTA Jacobi eigensolver vs cuSOLVER syevd inside the same solver build."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import paper_2302_12528_b200 as mp
from conftest import load_golden
names = sys.argv[1:] or ["lap3d8-dlobpcg-dchol", "lap3d16-dlobpcg-dchol", "lap3d16-mplobpcg-schol", "cfg1-dlobpcg-dchol", "cfg1-mplobpcg-schol", "dense256-dlobpcg-dchol"]
for name in names:
    g = load_golden(name)
    out = []
    for backend in (0, 1):
        ctx = mp.Context(0)
        ctx.set_option("spec_mode", 0)
        ctx.set_option("eig_backend", backend)
        from test_gpu_solver import make_op
        import test_gpu_solver as tg
        A = tg.make_op(mp, name) if False else None
        dims = {"lap3d8": (8,), "lap3d16": (16,), "cfg1": (32,)}
        key = name.split("-")[0]
        if key in dims:
            A = mp.laplace3d(*dims[key], ctx=ctx)
        else:
            from problems import spd_dense
            A = mp.dense_matrix(spd_dense(256, 1e3, 5)[0], ctx=ctx)
        cfg = mp.SolverConfig(variant=str(g["variant"]), **eval(str(g["kw"])))
        r = mp.solve(A, cfg)
        out.append(f"{r.iterations_lower}+{r.iterations_working}")
    print(f"{name:26s} jacobi {out[0]:>10s}  cusolver {out[1]:>10s}  ref {int(g['iters_lower'])}+{int(g['iters_working'])}", flush=True)
