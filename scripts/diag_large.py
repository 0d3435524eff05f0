"""Progress trace of one large solve (GPU box helper): prints every `every`-th
iteration record live and the last records when the solve throws.
python scripts/diag_large.py N k m variant every"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2302_12528_b200 as mp  # noqa: E402
from paper_2302_12528_b200 import api  # noqa: E402

N, k, m = (int(x) for x in sys.argv[1:4])
variant = sys.argv[4] if len(sys.argv) > 4 else "mplobpcg-schol"
every = int(sys.argv[5]) if len(sys.argv) > 5 else 200
t0 = time.time()
orig = api._History.__init__


def init(self):
    orig(self)
    inner = self.cb

    def sink(user, rec_p):
        inner(user, rec_p)
        i = len(self.records) - 1
        r = self.records[-1]
        if i % every == 0:
            rn = np.array(r.residual_norms[:k])
            print(f"{time.time() - t0:8.1f}s it {i:6d} st {r.stage} n_c {r.n_converged:3d} "
                  f"res {rn.max():.3e} drop {r.w_columns_dropped} rot {r.basis_rotation_fallback} "
                  f"th_k {r.ritz_values[k - 1]:.12e}", flush=True)
    self.cb = mp._lib.SINK(sink) if hasattr(mp, "_lib") else api.L.SINK(sink)
    self._keep = sink


api._History.__init__ = init
A = mp.laplace3d(N)
cfg = mp.SolverConfig(k=k, block=m, tol=1e-10, maxit=20000, variant=variant)
try:
    if os.environ.get("PREPARED"):  # bench.py's path: device-resident raw inputs
        import torch
        n, sr = A.n, cfg.sketch_rows
        X0 = torch.from_numpy(np.ascontiguousarray(mp.gaussian_matrix(n, m, cfg.seed).T)).cuda()
        Omh = mp.gaussian_matrix(n, sr, cfg.seed ^ 0x9E3779B97F4A7C15)
        Om = torch.from_numpy(np.ascontiguousarray(Omh.T)).cuda()
        fro = float(np.sqrt(np.sum(np.abs(Omh.ravel(order="F")) ** 2)))  # as bench.py
        for rep in range(int(os.environ.get("PREPARED"))):
            r = mp.solve_prepared(A, cfg, X0, Om, fro, T=mp.jacobi(A, mp.build_precision_for(variant)),
                                  history=True)
            print("rep", rep, r.converged, r.iterations_lower, r.iterations_working, flush=True)
    else:
        r = mp.solve(A, cfg, want_X=False)
    print("done", r.converged, r.iterations_lower, r.iterations_working, f"{time.time() - t0:.1f}s")
except Exception as e:
    print("EXC", type(e).__name__, e, f"{time.time() - t0:.1f}s")
