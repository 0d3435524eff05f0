"""One binary32 Gram G = A^T B at a solver shape (ncu target):
    python scripts/tc_gram_one.py [n] [ka] [kb] [reps]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 * 1024 * 1024
ka = int(sys.argv[2]) if len(sys.argv) > 2 else 240
kb = int(sys.argv[3]) if len(sys.argv) > 3 else 240
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ctx = mp.default_context()
import os  # noqa: E402
for kv in filter(None, os.environ.get("MPEIG_OPTS", "").split(",")):
    key, val = kv.split("=")
    assert ctx.lib.mpeig_set_process_option(key.encode(), int(val)) == 0, kv
A = torch.randn(ka, n, device="cuda")
B = torch.randn(kb, n, device="cuda")
G = torch.empty(kb, ka, device="cuda")
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for _ in range(reps):
    ctx.check(ctx.lib.mpeig_gram_f32(ctx.h, n, ka, p(A), n, kb, p(B), n, p(G)))
torch.cuda.synchronize()
print("ok", n, ka, kb)
