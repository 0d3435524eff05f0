import ctypes as C, sys, torch, numpy as np
sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp
ctx = mp.default_context()
n, k, c = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(0)
A = rng.standard_normal((n, k)).astype(np.float32); Cm = rng.standard_normal((k, c)).astype(np.float32)
Z = rng.standard_normal((n, c)).astype(np.float32)
dev = lambda M: torch.from_numpy(np.ascontiguousarray(M.T)).cuda()
Ad, Cd = dev(A), dev(Cm)
Yr = A.astype(np.float64) @ Cm.astype(np.float64)
import os
for stage, depth in ((1, 0),):
    ctx.lib.mpeig_set_process_option(b"tc_stage", stage)
    ctx.lib.mpeig_set_process_option(b"g2_depth", depth)
    for beta, inplace in ((0.0, False), (1.0, False), (1.0, True)):
        Zd = dev(Z); Yd = Zd if inplace else torch.zeros_like(Zd)
        ctx.check(ctx.lib.mpeig_gemm_f32(ctx.h, n, k, c, 1.0, C.c_void_p(Ad.data_ptr()), n, C.c_void_p(Cd.data_ptr()), k, beta, C.c_void_p(Zd.data_ptr()), n, C.c_void_p(Yd.data_ptr()), n))
        Y = Yd.cpu().numpy().T.astype(np.float64)
        err = np.abs(Y - (Yr + beta * Z))
        bad = np.argwhere(err > 1e-3)
        print(f"stage={stage} depth={depth} beta={beta} inplace={inplace}: max err {err.max():.3e}  bad {len(bad)}  first {bad[:5].tolist()}  rows {np.unique(bad[:,0]//128)[:10].tolist() if len(bad) else []} cols {np.unique(bad[:,1])[:20].tolist() if len(bad) else []}", flush=True)
ctx.lib.mpeig_set_process_option(b"tc_stage", 1)
import os
ctx.lib.mpeig_set_process_option(b"tc_ablate", int(os.environ.get("ABL", "0")))
Yd = torch.zeros_like(dev(Z))
ctx.check(ctx.lib.mpeig_gemm_f32(ctx.h, n, k, c, 1.0, C.c_void_p(Ad.data_ptr()), n, C.c_void_p(Cd.data_ptr()), k, 0.0, None, 0, C.c_void_p(Yd.data_ptr()), n))
Y = Yd.cpu().numpy().T.astype(np.float64)
print("Y[0:3,0:3]", Y[0:3, 0:3].round(3).tolist())
print("Yr[0:3,0:3]", Yr[0:3, 0:3].round(3).tolist())
# locate where Y's first tile came from
for r0 in range(0, n, 128):
    if np.allclose(Y[0:128], Yr[r0:r0 + 128], atol=1e-3):
        print("Y tile 0 == Yr tile", r0 // 128)
for r0 in range(0, n - 127, 128):
    if np.allclose(Yr[0:128], Y[r0:r0 + 128], atol=1e-3):
        print("Yr tile 0 found at Y tile", r0 // 128)
print("zeros in Y:", int((Y == 0).sum()), "of", Y.size)
ok_rows = np.all(np.abs(Y - Yr) < 1e-3, axis=1)
print("correct rows:", int(ok_rows.sum()), "tiles fully correct:", [t for t in range(n // 128) if ok_rows[t*128:(t+1)*128].all()][:20])
ok_cols = np.all(np.abs(Y - Yr) < 1e-3, axis=0)
print("correct cols:", np.nonzero(ok_cols)[0][:40].tolist())
print("Y[200,:8]", Y[200, :8].round(3).tolist()); print("Yr[200,:8]", Yr[200, :8].round(3).tolist())
# is Y a permutation of entries of Yr?  match Y[200,0] anywhere
v = Y[200, 0]
loc = np.argwhere(np.abs(Yr - v) < 1e-4)
print("Y[200,0] found in Yr at", loc[:5].tolist())
v = Y[200, 1]
loc = np.argwhere(np.abs(Yr - v) < 1e-4)
print("Y[200,1] found in Yr at", loc[:5].tolist())
bad = np.abs(Y - Yr) > 1e-3
for t in range(min(4, n // 128)):
    b = bad[t*128:(t+1)*128]
    print(f"tile {t}: bad {int(b.sum())}  bad rows {np.nonzero(b.any(1))[0][:8].tolist()}..  bad cols {np.nonzero(b.any(0))[0][:8].tolist()}..")
    # source of Y rows in this tile
    for r in (0, 40, 72, 127):
        rr = t*128 + r
        src = [int(q) for q in np.nonzero(np.all(np.abs(Yr - Y[rr]) < 1e-3, axis=1))[0][:3]]
        print(f"   Y row {rr} == Yr rows {src}  zero={bool(np.all(Y[rr]==0))}")
