"""Iteration count of one golden case under the solver's execution / eigensolver
options (GPU box helper): python scripts/ab_variants.py dense256-dlobpcg-dchol"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2302_12528_b200 as mp  # noqa: E402
from conftest import load_golden  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "dense256-dlobpcg-dchol"
g = load_golden(name)
kw = eval(str(g["kw"]))
print(name, "ref", int(g["iters_lower"]), int(g["iters_working"]))
opts = [{}, {"ql_exact": 1}, {"ql_exact": 3}, {"ql_exact": 2}, {"spec_mode": 0}, {"eig_backend": 1},
        {"eig_backend": 2}]
for o in opts:
    ctx = mp.Context(0)
    for k, v in o.items():
        ctx.set_option(k, v)
    # operators must live on the context that solves
    if name.startswith("dense256"):
        from problems import spd_dense
        A = mp.dense_matrix(spd_dense(256, 1e3, 5)[0], ctx=ctx)
    elif name.startswith("cfg1"):
        A = mp.laplace3d(32, ctx=ctx)
    elif name.startswith("lap3d16"):
        A = mp.laplace3d(16, ctx=ctx)
    elif name.startswith("lap3d8"):
        A = mp.laplace3d(8, ctx=ctx)
    r = mp.solve(A, mp.SolverConfig(variant=str(g["variant"]), **kw))
    print(o, r.iterations_lower, r.iterations_working, r.converged, flush=True)
