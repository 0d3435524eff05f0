import os, sys, ctypes as C
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np, torch
import paper_2302_12528_b200 as mp
os.environ["MPEIG_DUMP_G_ITER"] = "280"
os.environ["MPEIG_DUMP_G_FILE"] = "gpurun_out/G280.bin"
ctx = mp.Context(0); ctx.set_option("spec_mode", 0); ctx.set_option("eig_backend", 1)
A = mp.laplace3d(16, ctx=ctx)
r = mp.solve(A, mp.SolverConfig(variant="dlobpcg-dchol", k=10, block=16, tol=1e-10, maxit=2000))
G = np.fromfile("gpurun_out/G280.bin").reshape(48, 48).T
print("G sym dev", np.abs(G - G.T).max(), "norm", np.linalg.norm(G))
lam, V = np.linalg.eigh(G)
for backend in (0, 1):
    ctx.set_option("eig_backend", backend)
    Md = mp.to_device(G)
    vals = torch.zeros(48, dtype=torch.float64, device="cuda"); vecs = torch.zeros((48, 48), dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.mpeig_small_eig_f64(ctx.h, 48, C.c_void_p(Md.data_ptr()), C.c_void_p(vals.data_ptr()), C.c_void_p(vecs.data_ptr())))
    v = vals.cpu().numpy(); Vd = mp.to_host(vecs)
    res = np.linalg.norm(G @ Vd - Vd * v, axis=0)
    print("backend", backend, "eig err max", np.abs(v - lam).max(), "orth", np.abs(Vd.T @ Vd - np.eye(48)).max())
    print("   resid per col (first 16)", np.array2string(res[:16], precision=1))
    print("   X-components of P cols |C(0:16,16:32)| colnorms", np.array2string(np.linalg.norm(Vd[:16, 16:32], axis=0), precision=2))
print("lam", lam[:20])
