import ctypes as C, sys, torch, numpy as np
sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp
ctx = mp.default_context()
import os
for kv in filter(None, os.environ.get("MPEIG_OPTS", "").split(",")):
    key, val = kv.split("=")
    assert ctx.lib.mpeig_set_process_option(key.encode(), int(val)) == 0, kv
rng = np.random.default_rng(0)
for n, ka, kb in ((32, 48, 48), (64, 144, 144), (4096, 48, 48), (4096, 240, 240), (65536, 80, 80)):
    A = rng.standard_normal((n, ka)).astype(np.float32)
    B = rng.standard_normal((n, kb)).astype(np.float32)
    Ad = torch.from_numpy(np.ascontiguousarray(A.T)).cuda(); Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    Gr = A.astype(np.float64).T @ B.astype(np.float64)
    sc = np.abs(A).astype(np.float64).T @ np.abs(B).astype(np.float64)
    res = []
    for opt in (2, 0):
        ctx.lib.mpeig_set_process_option(b"gram_tc", opt)
        Gd = torch.zeros((kb, ka), dtype=torch.float32, device="cuda")
        ctx.check(ctx.lib.mpeig_gram_f32(ctx.h, n, ka, C.c_void_p(Ad.data_ptr()), n, kb, C.c_void_p(Bd.data_ptr()), n, C.c_void_p(Gd.data_ptr())))
        G = Gd.cpu().numpy().T.astype(np.float64)
        res.append(np.max(np.abs(G - Gr) / sc))
    print(f"gram n={n} {ka}x{kb}: max |err|/(|A|^T|B|)  TC {res[0]:.2e}  SIMT {res[1]:.2e}  (u32 {2**-24:.1e})", flush=True)
for n, k, c in ((128, 16, 16), (4096, 48, 48), (4096, 80, 80), (65536, 240, 160), (8192, 576, 384)):
    A = rng.standard_normal((n, k)).astype(np.float32); Cm = rng.standard_normal((k, c)).astype(np.float32)
    Ad = torch.from_numpy(np.ascontiguousarray(A.T)).cuda(); Cd = torch.from_numpy(np.ascontiguousarray(Cm.T)).cuda()
    Yr = A.astype(np.float64) @ Cm.astype(np.float64); sc = np.abs(A).astype(np.float64) @ np.abs(Cm).astype(np.float64)
    res = []
    for opt in (2, 0):
        ctx.lib.mpeig_set_process_option(b"gemm_tc", opt)
        Yd = torch.zeros((c, n), dtype=torch.float32, device="cuda")
        ctx.check(ctx.lib.mpeig_gemm_f32(ctx.h, n, k, c, 1.0, C.c_void_p(Ad.data_ptr()), n, C.c_void_p(Cd.data_ptr()), k, 0.0, None, 0, C.c_void_p(Yd.data_ptr()), n))
        Y = Yd.cpu().numpy().T.astype(np.float64)
        res.append((np.max(np.abs(Y - Yr) / sc), np.sqrt(np.mean((np.abs(Y - Yr) / sc) ** 2))))
    ctx.lib.mpeig_set_process_option(b"gemm_tc", 1)
    print(f"gemm n={n} k={k} c={c}: max/rms |err|/(|A||C|)  TC {res[0][0]:.2e}/{res[0][1]:.2e}  "
          f"SIMT {res[1][0]:.2e}/{res[1][1]:.2e}", flush=True)
