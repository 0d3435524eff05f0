"""One binary32 block update Y = A C at a solver shape (ncu target):
    python scripts/tc_gemm_one.py [n] [k] [c] [reps]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 * 1024 * 1024
k = int(sys.argv[2]) if len(sys.argv) > 2 else 240
c = int(sys.argv[3]) if len(sys.argv) > 3 else 160
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ctx = mp.default_context()
import os  # noqa: E402
for kv in filter(None, os.environ.get("MPEIG_OPTS", "").split(",")):
    key, val = kv.split("=")
    assert ctx.lib.mpeig_set_process_option(key.encode(), int(val)) == 0, kv
A = torch.randn(k, n, device="cuda")
Cm = torch.randn(c, k, device="cuda")
Y = torch.empty(c, n, device="cuda")
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for _ in range(reps):
    ctx.check(ctx.lib.mpeig_gemm_f32(ctx.h, n, k, c, 1.0, p(A), n, p(Cm), k, 0.0, None, 0, p(Y), n))
torch.cuda.synchronize()
print("ok", n, k, c)
