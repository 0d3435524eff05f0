"""Rounding sensitivity of the REFERENCE algorithm's iteration counts.

Builds the plain-C restatement (oracle/mp_oracle.c -- bitwise identical to the
reference, tests/test_oracle.py) a second time with FMA contraction
(-ffp-contract=fast -mfma): same algorithm, same operation order, only the
rounding of a*b+c changes.  The iteration counts it needs on the golden cases
quantify how much the reference's own iteration count moves under
rounding-level perturbations; tests/test_gpu_solver.py uses this band for the
GPU path, whose reductions necessarily round differently.

    python tests/golden/make_sensitivity.py [--variant=fma|reassoc] [case ...]
        -> tests/golden/sensitivity.json
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from oracle import Oracle  # noqa: E402
from golden.make_golden import CASES  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "sensitivity.json")
# rounding-only perturbations of the same algorithm and operation sequence:
#   fma      a*b+c contracted (one rounding instead of two)
#   reassoc  FMA plus reassociated, vectorised reductions (different summation
#            order in dot products and Gram sums -- what a parallel device does)
#   jacobi   the Rayleigh-Ritz eigendecomposition by cyclic Jacobi instead of
#            tridiagonal QL: a different valid eigensolver, i.e. a different
#            rounding of the Ritz vectors (the GPU's eigensolver runs the
#            reference's QL but rounds differently)
VARIANTS = {
    "jacobi": ["-DMPORC_EIG_JACOBI"],
    "fma": ["-ffp-contract=fast", "-mfma"],
    "reassoc": ["-ffp-contract=fast", "-mfma", "-mavx2", "-fassociative-math", "-fno-signed-zeros",
                "-fno-trapping-math"],
}


def build(variant):
    lib = f"/tmp/liboracle_{variant}.so"
    src = os.path.join(ROOT, "oracle", "mp_oracle.c")
    subprocess.run(["gcc", "-std=c11", "-O3", "-DNDEBUG", "-fPIC", *VARIANTS[variant], "-shared", "-o",
                    lib, src, "-lm"], check=True)
    return lib


def main():
    args = sys.argv[1:]
    which = list(VARIANTS)
    if args and args[0].startswith("--variant="):
        which = [args.pop(0).split("=", 1)[1]]
    names = args or [n for n in CASES if not n.startswith("cfg1")]
    for v in which:
        orc = Oracle("port")
        orc.lib = C.CDLL(build(v))
        for name in names:
            make, variant, kw = CASES[name]
            r = orc.solve(make(), variant, **kw)
            # re-read before writing: several of these may run side by side
            data = json.load(open(OUT)) if os.path.exists(OUT) else {}
            e = data.setdefault(name, {})
            e[f"{v}_iters_lower"] = r.iters_lower
            e[f"{v}_iters_working"] = r.iters_working
            e[f"{v}_converged"] = r.converged
            print(v, name, e, flush=True)
            json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
