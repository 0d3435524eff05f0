import ctypes as C, sys, torch, json
sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp
ctx = mp.default_context()
n = 2097152
out = []
for ka in (48, 240):
    A = torch.randn(ka, n, dtype=torch.float32, device="cuda")
    G = torch.zeros(ka, ka, dtype=torch.float32, device="cuda")
    for nprod, st in ((8, 1), (1, 1), (8, 0), (1, 0), (0, 1)):
        ctx.lib.mpeig_set_process_option(b"gram_tc", 2)
        ctx.lib.mpeig_set_process_option(b"tc_nprod", nprod)
        ctx.lib.mpeig_set_process_option(b"tc_store", st)
        f = lambda: ctx.check(ctx.lib.mpeig_gram_f32(ctx.h, n, ka, C.c_void_p(A.data_ptr()), n, ka, C.c_void_p(A.data_ptr()), n, C.c_void_p(G.data_ptr())))
        f(); torch.cuda.synchronize()
        with mp.profile():
            for _ in range(3): f()
            torch.cuda.synchronize()
            r = mp.profile.report()["gram_f32"]
        out.append((ka, nprod, st, r["ms"] / r["count"]))
        print(out[-1], flush=True)
