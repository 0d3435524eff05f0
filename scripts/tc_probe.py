"""Run the binary32 tensor-core Gram once at a given shape (ncu target)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp  # noqa: E402

n, ka, kb = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (2097152, 240, 240)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ctx = mp.default_context()
assert ctx.lib.mpeig_set_process_option(b"gram_tc", 2) == 0
A = torch.randn(ka, n, dtype=torch.float32, device="cuda")
B = torch.randn(kb, n, dtype=torch.float32, device="cuda")
G = torch.zeros(kb, ka, dtype=torch.float32, device="cuda")
for _ in range(reps):
    ctx.check(ctx.lib.mpeig_gram_f32(ctx.h, n, ka, C.c_void_p(A.data_ptr()), n, kb,
                                     C.c_void_p(B.data_ptr()), n, C.c_void_p(G.data_ptr())))
torch.cuda.synchronize()
print("ok")
