"""Iteration-count envelope of the REFERENCE under rounding-level input noise.

LOBPCG iteration counts on these spectra are a chaotic function of rounding
(degenerate eigenvalue clusters, the prefix convergence rule, the fp32 stage's
exit near its attainable accuracy).  This script measures how far the
unmodified reference itself (oracle/_ref, built from /root/reference) moves when
its start block is perturbed by at most one binary64 ulp per entry
(tests/problems.py::perturb_x0, p = 1..NPERT), per stage.  The device is held
to that envelope (tests/test_gpu_solver.py) instead of a fixed percentage band.

    python tests/golden/make_envelope.py                 # the fast cases
    python tests/golden/make_envelope.py --case cfg1-mplobpcg-schol -j 6

Output: tests/golden/envelope.json  {case: {"ref": [lower, working],
"perturbed": [[lower, working], ...], "npert": N}}
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.dirname(os.path.abspath(__file__))]

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "envelope.json")
NPERT = 16

# callback-harness cases of make_golden.py (the stock-driver "native" cases draw
# their start block inside the reference and cannot take a perturbed X0)
FAST = ["lap3d8-dlobpcg-dchol", "lap3d8-dlobpcg-schol", "lap3d8-mplobpcg-schol", "lap3d8-pinvit",
        "lap3d16-dlobpcg-dchol", "lap3d16-dlobpcg-schol", "lap3d16-mplobpcg-schol",
        "lap2d50-mplobpcg-schol", "lap2d50-dlobpcg-dchol", "lap2d5x500-mplobpcg-schol",
        "dense256-dlobpcg-dchol", "dense256-mplobpcg-schol", "lap2d32-pinvit"]
SLOW = ["cfg1-mplobpcg-schol", "cfg1-dlobpcg-dchol", "cfg1-dlobpcg-schol"]
# the large-block path (3m = 144 > 96)
LARGE = ["lap2d64k32-dlobpcg-dchol", "lap2d64k32-mplobpcg-schol", "lap2d128k32-dlobpcg-dchol",
         "ks32-dlobpcg-dchol", "ks32-mplobpcg-schol"]


def one(args):
    name, p = args
    from make_golden import CASES
    from oracle import Oracle
    from problems import envelope_ulp, perturb_x0
    make, variant, kw = CASES[name]
    prob = make()
    kw = dict(kw)
    k = kw["k"]
    m = kw.get("block") or (3 * k + 1) // 2
    o = Oracle("ref")
    x0 = perturb_x0(o.gaussian(prob.n, m, kw.get("seed", 0)), p, envelope_ulp(variant))
    r = o.solve(prob, variant, x0=x0, hist_cap=0, **kw)
    return name, p, int(r.iters_lower), int(r.iters_working), bool(r.converged), r.status


def CASES_VARIANT(name):
    from make_golden import CASES
    return CASES[name][1]


def main():
    from problems import envelope_ulp
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append")
    ap.add_argument("-j", type=int, default=6)
    ap.add_argument("--npert", type=int, default=NPERT)
    a = ap.parse_args()
    cases = a.case or FAST
    env = json.load(open(OUT)) if os.path.exists(OUT) else {}
    jobs = [(c, p) for c in cases for p in range(0, a.npert + 1)]
    res = {c: {} for c in cases}
    with ProcessPoolExecutor(a.j) as ex:
        for name, p, lo, wk, conv, st in ex.map(one, jobs):
            res[name][p] = (lo, wk, conv, st)
            print(f"{name} p={p}: {lo}+{wk} conv={conv} status={st}", flush=True)
    env = json.load(open(OUT)) if os.path.exists(OUT) else {}  # merge with concurrent runs
    for c in cases:
        r = res[c]
        env[c] = {"ref": list(r[0][:2]), "npert": a.npert,
                  "perturbed": [list(r[p][:2]) for p in range(1, a.npert + 1)],
                  "converged": [bool(r[p][2]) for p in range(0, a.npert + 1)],
                  "ulp": envelope_ulp(CASES_VARIANT(c))}
        env = dict(sorted(env.items()))
        with open(OUT, "w") as f:
            json.dump(env, f, indent=1)


if __name__ == "__main__":
    main()
