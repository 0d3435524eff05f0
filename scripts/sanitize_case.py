"""Small end-to-end workload for compute-sanitizer (tests/test_gpu_sanitizer.py):
LOBPCG on lap3d 8^3 in working and mixed precision (speculative body, CUDA graph,
last-CTA tickets, one-CTA eigensolver), PINVIT, and the tcgen05 binary32 Gram /
block update forced on small shapes."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp  # noqa: E402

tools = sys.argv[1] if len(sys.argv) > 1 else "all"
A = mp.laplace3d(8)
for variant in ("dlobpcg-dchol", "mplobpcg-schol", "pinvit"):
    cfg = mp.SolverConfig(k=4, tol=1e-8, maxit=60, variant=variant)
    r = mp.solve(A, cfg)
    print(variant, r.iterations_lower, r.iterations_working, flush=True)
import torch  # noqa: E402
ctx = mp.default_context()
ctx.lib.mpeig_set_process_option(b"tc", 2)
n, ka = 300, 40
X = torch.randn(ka, n, dtype=torch.float32, device="cuda")
G = torch.zeros(ka, ka, dtype=torch.float32, device="cuda")
ctx.check(ctx.lib.mpeig_gram_f32(ctx.h, n, ka, C.c_void_p(X.data_ptr()), n, ka,
                                 C.c_void_p(X.data_ptr()), n, C.c_void_p(G.data_ptr())))
Y = torch.zeros(ka, n, dtype=torch.float32, device="cuda")
ctx.check(ctx.lib.mpeig_gemm_f32(ctx.h, n, ka, ka, 1.0, C.c_void_p(X.data_ptr()), n,
                                 C.c_void_p(G.data_ptr()), ka, 0.0, None, 0, C.c_void_p(Y.data_ptr()), n))
torch.cuda.synchronize()
ctx.lib.mpeig_set_process_option(b"tc", 1)
print("ok", float(np.abs(G.cpu().numpy()).max()))
