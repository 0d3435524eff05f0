"""The C++ drop-in layer (include/mpeig_b200.hpp) against the reference.

tests/cpp/dropin_main.cpp is compiled against the reference's OWN headers
(/root/reference/proj/include) and linked to libmpeig_b200.so by
oracle/Makefile (`make -C oracle dropin`, also run by __graft_entry__.build()),
so the reference's types, BlockOperator callbacks and call sequences run the
B200 path unchanged: the CPU test checks that the header compiles and links
against the reference; the GPU tests run the reference's run_variant flow
(drivers.hpp:79-108) with every lobpcg_stage qualified as
mpeig::b200::lobpcg_stage, and the stock drivers solve(CsrMatrix) /
solve(DenseMatrix) through the header, against the golden fixtures.
"""
import json
import os
import subprocess
import types

import numpy as np
import pytest

from conftest import ROOT, load_golden

BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_main")
REF_INCLUDE = "/root/reference/proj/include/mpeig/eigensolvers.hpp"


def test_dropin_header_builds_against_reference():
    if not os.path.exists(REF_INCLUDE):
        if os.path.exists(BIN):
            return  # prebuilt where the reference was present
        pytest.skip("reference sources absent and no prebuilt drop-in driver")
    lib = os.path.join(ROOT, "paper_2302_12528_b200", "libmpeig_b200.so")
    if not os.path.exists(lib):
        pytest.skip("libmpeig_b200.so not built")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"], check=True)
    assert os.path.exists(BIN)


def run(*args):
    if not os.path.exists(BIN):
        pytest.skip("drop-in driver not built (make -C oracle dropin)")
    p = subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.stdout, p.stderr)
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert "error" not in d, d
    return d


def as_result(d, k):
    return types.SimpleNamespace(
        theta=np.array(d["theta"][:k]), converged=d["converged"],
        iterations_lower=d["iters_lower"], iterations_working=d["iters_working"],
        a_norm_estimate=d["a_norm_est"], residual_norms=np.zeros(k))


def check(name, d, slack=None):
    from test_gpu_solver import check_parity
    g = load_golden(name)
    kw = eval(str(g["kw"]))
    cfg = types.SimpleNamespace(tol=kw["tol"], k=kw["k"])
    check_parity(g, cfg, as_result(d, kw["k"]), name, iter_slack=slack)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["dlobpcg-dchol", "dlobpcg-schol", "mplobpcg-schol"])
def test_dropin_lobpcg_stage_lap3d8(variant):
    """run_variant's flow with the reference's CPU callbacks, lobpcg_stage on the B200."""
    d = run("stage", 8, 8, 8, variant, 4, 1e-10, 500)
    check(f"lap3d8-{variant}", d)
    stages = 2 if variant == "mplobpcg-schol" else 1
    assert d["history"] == d["iters_lower"] + d["iters_working"] + stages


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["dlobpcg-dchol", "dlobpcg-schol", "mplobpcg-schol"])
def test_dropin_solve_csr(variant):
    """mpeig::b200::solve(CsrMatrix) == the reference's stock sparse driver."""
    from test_gpu_spchol import _band
    name = f"splap3d16-{variant}"
    d = run("solve_csr", 16, 16, 16, variant, 10, 16, 1e-10, 500, 0)
    check(name, d, slack=_band(name))
    assert d["precond_shift"] == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["dlobpcg-dchol", "mplobpcg-schol"])
def test_dropin_solve_dense(variant, tmp_path):
    """mpeig::b200::solve(DenseMatrix) == the reference's stock dense driver."""
    from problems import spd_dense
    A = spd_dense(256, 1e3, 5)[0]
    f = tmp_path / "a.bin"
    np.asfortranarray(A).ravel(order="F").tofile(f)
    d = run("solve_dense", f, 256, variant, 8, 1e-10, 500, 3)
    check(f"dense256chol-{variant}", d, slack=2)


@pytest.mark.gpu
def test_dropin_exceptions():
    """ConfigError, NotPositiveDefinite and a callback's DimensionMismatch come
    out of the B200 path as the reference's own exception types."""
    d = run("errors")
    assert d["ok"] == d["total"] == 3
