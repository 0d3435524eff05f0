"""Rounding sensitivity of the REFERENCE algorithm's iteration counts.

Builds the plain-C restatement (oracle/mp_oracle.c -- bitwise identical to the
reference, tests/test_oracle.py) a second time with FMA contraction
(-ffp-contract=fast -mfma): same algorithm, same operation order, only the
rounding of a*b+c changes.  The iteration counts it needs on the golden cases
quantify how much the reference's own iteration count moves under
rounding-level perturbations; tests/test_gpu_solver.py uses this band for the
GPU path, whose reductions necessarily round differently.

    python tests/golden/make_sensitivity.py [case ...]   -> tests/golden/sensitivity.json
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
FMA_LIB = "/tmp/liboracle_fma.so"


def build_fma():
    src = os.path.join(ROOT, "oracle", "mp_oracle.c")
    subprocess.run(["gcc", "-std=c11", "-O3", "-DNDEBUG", "-fPIC", "-ffp-contract=fast", "-mfma",
                    "-shared", "-o", FMA_LIB, src, "-lm"], check=True)


def main():
    build_fma()
    orc = Oracle("port")
    orc.lib = C.CDLL(FMA_LIB)
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    names = sys.argv[1:] or [n for n in CASES if not n.startswith("cfg1")]
    for name in names:
        make, variant, kw = CASES[name]
        r = orc.solve(make(), variant, **kw)
        data[name] = {"fma_iters_lower": r.iters_lower, "fma_iters_working": r.iters_working,
                      "fma_converged": r.converged}
        print(name, data[name], flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
