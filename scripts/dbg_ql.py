import os, sys, ctypes as C
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np, torch
import paper_2302_12528_b200 as mp
ctx = mp.Context(0)
G = np.fromfile("build/G280.bin").reshape(48, 48).T
lam = np.linalg.eigvalsh(G)
for meth in (0, 1, 2, 3):
    ctx.set_option("syev_method", meth)
    Md = mp.to_device(G)
    vals = torch.zeros(48, dtype=torch.float64, device="cuda"); vecs = torch.zeros((48, 48), dtype=torch.float64, device="cuda")
    rc = ctx.lib.mpeig_small_eig_f64(ctx.h, 48, C.c_void_p(Md.data_ptr()), C.c_void_p(vals.data_ptr()), C.c_void_p(vecs.data_ptr()))
    v = vals.cpu().numpy(); V = mp.to_host(vecs)
    print(meth, "rc", rc, "eig err", np.abs(v - lam).max(), "orth", np.abs(V.T @ V - np.eye(48)).max(), "res", np.abs(G @ V - V * v).max())
# a random symmetric matrix and a diagonal-dominant one
for name, M in (("rand", (lambda X: X + X.T)(np.random.default_rng(1).standard_normal((48, 48)))),
                ("diagdom", np.diag(np.arange(48.0)) + 1e-12 * (lambda X: X + X.T)(np.random.default_rng(2).standard_normal((48, 48)))),
                ("degenerate", np.diag(np.repeat([1.0, 2.0, 3.0, 4.0], 12)) + 1e-9 * (lambda X: X + X.T)(np.random.default_rng(3).standard_normal((48, 48))))):
    ctx.set_option("syev_method", 0)
    Md = mp.to_device(M)
    vals = torch.zeros(48, dtype=torch.float64, device="cuda"); vecs = torch.zeros((48, 48), dtype=torch.float64, device="cuda")
    rc = ctx.lib.mpeig_small_eig_f64(ctx.h, 48, C.c_void_p(Md.data_ptr()), C.c_void_p(vals.data_ptr()), C.c_void_p(vecs.data_ptr()))
    v = vals.cpu().numpy(); V = mp.to_host(vecs)
    print(name, "rc", rc, "eig err", np.abs(v - np.linalg.eigvalsh(M)).max(), "orth", np.abs(V.T @ V - np.eye(48)).max())
