import sys, time, torch
sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp
ctx = mp.default_context()
A = mp.laplace3d(32)
cfg = mp.SolverConfig(k=10, block=16, tol=1e-10, maxit=2000, variant="mplobpcg-schol")
for ch in [int(x) for x in sys.argv[1:]]:
    ctx.lib.mpeig_set_process_option(b"gram_chunks", ch)
    mp.solve(A, cfg, want_X=False, history=False)
    torch.cuda.synchronize(); t = time.perf_counter()
    r = mp.solve(A, cfg, want_X=False, history=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    its = r.iterations_lower + r.iterations_working
    print(f"chunks {ch}: {r.iterations_lower}+{r.iterations_working} {dt:.4f} s  {1e6*dt/its:.1f} us/it", flush=True)
