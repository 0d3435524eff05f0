import sys
sys.path[:0] = [__file__.rsplit("/scripts/", 1)[0], __file__.rsplit("/scripts/", 1)[0] + "/tests"]
import paper_2302_12528_b200 as mp
from test_gpu_solver import run_case
ctx = mp.default_context()
for name in ("lap3d16-mplobpcg-schol", "lap3d8-mplobpcg-schol"):
    for key, val in (("tc", 0), ("gram_tc", 2), ("gemm_tc", 2), ("tc", 2)):
        ctx.lib.mpeig_set_process_option(b"tc", 0)
        ctx.lib.mpeig_set_process_option(key.encode(), val)
        g, cfg, r = run_case(mp, name)
        print(name, key, val, r.iterations_lower, r.iterations_working, "ref", int(g["iters_lower"]), int(g["iters_working"]), flush=True)
