"""Row-sharded solve with ranks as threads (host-staged exchanges) vs one GPU.
GPU box helper: python scripts/shard_demo.py [nranks] [n]"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_12528_b200 as mp  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 16
for variant in ("dlobpcg-dchol", "mplobpcg-schol"):
    cfg = mp.SolverConfig(k=10, block=16, tol=1e-10, maxit=2000, variant=variant)
    A1 = mp.laplace3d(N)
    t = time.time()
    r1 = mp.solve(A1, cfg)
    t1 = time.time() - t
    group = mp.HostGroup(P)
    sl = mp.slab_partition(N, P)
    out = [None] * P

    def work(r):
        ctx = mp.Context(0, stream=torch.cuda.Stream())
        ctx.attach_host(group, r)
        A = mp.laplace3d_slab(N, N, N, sl[r][0], sl[r][1], ctx=ctx)
        out[r] = mp.solve(A, cfg)

    t = time.time()
    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    [x.start() for x in th]
    [x.join() for x in th]
    tp = time.time() - t
    rp = out[0]
    print(f"{variant} n={N}^3 ranks={P}: 1-GPU {r1.iterations_lower}+{r1.iterations_working} "
          f"({t1:.2f}s)  sharded {rp.iterations_lower}+{rp.iterations_working} ({tp:.2f}s, host-staged)  "
          f"max|dtheta|/theta {np.max(np.abs(rp.theta - r1.theta) / r1.theta):.1e}", flush=True)
