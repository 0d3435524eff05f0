"""Per-iteration cost at a large configuration (GPU box helper):
python scripts/large_iter.py [N] [k] [block] [iters] -> kernel shares of a capped solve."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2302_12528_b200 as mp  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
m = int(sys.argv[3]) if len(sys.argv) > 3 else 48
it = int(sys.argv[4]) if len(sys.argv) > 4 else 20
for variant in ("dlobpcg-dchol", "mplobpcg-schol"):
    A = mp.laplace3d(N)
    cfg = mp.SolverConfig(k=k, block=m, tol=1e-10, maxit=it, variant=variant)
    mp.solve(A, cfg, want_X=False, history=False)  # warm-up
    t = time.time()
    r = mp.solve(A, cfg, want_X=False, history=False)
    dt = time.time() - t
    its = r.iterations_lower + r.iterations_working
    print(f"{variant} n={N}^3 k={k} m={m}: {its} iterations in {dt:.3f} s -> {1e3 * dt / its:.2f} ms/iteration",
          flush=True)
    with mp.profile() as p:
        mp.solve(A, cfg, want_X=False, history=False)
    rep = p.report()
    tot = sum(v["ms"] for v in rep.values())
    for name, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])[:8]:
        print(f"   {name:14s} {v['count']:6d} launches  {v['ms'] / v['count'] * 1e3:9.1f} us/launch  "
              f"{100 * v['ms'] / tot:5.1f} %")
