"""Iteration counts of the GPU solver on every golden case vs the reference
and the reference's own per-stage envelope under 1-ulp start-block
perturbations (tests/golden/envelope.json).  GPU box helper:

    python scripts/golden_iters.py [name-substring ...]
    MPEIG_OPTS="spec_qr=0,..." selects execution options of the default context.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2302_12528_b200 as mp  # noqa: E402
from conftest import load_golden  # noqa: E402
from test_gpu_solver import iteration_bands, make_op  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
names = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f != "pcg64.npz")
flt = sys.argv[1:]
ctx = mp.default_context()
for kv in filter(None, os.environ.get("MPEIG_OPTS", "").split(",")):
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
for name in names:
    if flt and not any(s in name for s in flt):
        continue
    g = load_golden(name)
    kw = eval(str(g["kw"]))
    cfg = mp.SolverConfig(variant=str(g["variant"]), **kw)
    ctx.spec_rollbacks(reset=True)
    r = mp.solve(make_op(mp, name), cfg)
    rb = ctx.spec_rollbacks()
    ref = (int(g["iters_lower"]), int(g["iters_working"]))
    got = (r.iterations_lower, r.iterations_working)
    rel = float(np.max(np.abs(r.theta - g["theta"]) / np.abs(g["theta"])))
    bands = iteration_bands(name, g)
    ok = all(lo <= v <= hi for v, (lo, hi) in zip((*got, sum(got)), bands))
    print(f"{name:28s} ref {ref[0]:5d}+{ref[1]:5d}  gpu {got[0]:5d}+{got[1]:5d}  "
          f"bands lower {bands[0]} working {bands[1]} {'ok' if ok else 'OUT'}  theta {rel:.1e}  "
          f"rollbacks {rb}", flush=True)
