import os, sys, ctypes as C
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np, torch
os.environ["MPEIG_DUMP_G_ITER"] = "-1"
os.environ["MPEIG_DUMP_G_FILE"] = "gpurun_out/Gfail.bin"
import paper_2302_12528_b200 as mp
ctx = mp.Context(0); ctx.set_option("spec_mode", 0); ctx.set_option("syev_method", 0)
A = mp.laplace3d(16, ctx=ctx)
h = []
try:
    r = mp.solve(A, mp.SolverConfig(variant="dlobpcg-dchol", k=10, block=16, tol=1e-10, maxit=3000))
    print("ok", r.iterations_working)
except Exception as e:
    print("ERR", e)
G = np.fromfile("gpurun_out/Gfail.bin")
s = int(round(len(G) ** 0.5)); G = G.reshape(s, s).T
print("s", s, "finite", np.isfinite(G).all(), "sym", np.abs(G - G.T).max(), "norm", np.linalg.norm(G))
print("eigs", np.linalg.eigvalsh(G)[:8])
np.save("gpurun_out/Gfail.npy", G)
