"""Pin the CPU oracle (oracle/mp_oracle.c) before trusting it.

1. Known-answer vectors from the reference's own tests.
2. The restatement against the reference itself (oracle/_ref, same inputs),
   bit for bit where the reference is deterministic.
3. The restatement against the committed golden fixtures (produced by the
   reference, tests/golden/make_golden.py) -- these travel to the GPU box.
"""
import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import Oracle, Problem, available
from problems import spd_dense


@pytest.fixture(scope="module")
def port():
    return Oracle("port")


@pytest.fixture(scope="module")
def ref():
    if not available("ref"):
        pytest.skip("reference build (oracle/_ref) absent")
    return Oracle("ref")


# ------------------------------------------------------------ known answers
def test_pcg64_golden_outputs(port):
    """tests/test_precision.cpp:56-71 (independent big-integer implementation)."""
    assert [int(x) for x in port.pcg64(0, 4)] == [
        0x01070196E695F8F1, 0x703EC840C59F4493, 0xE54954914B3A44FA, 0x96130FF204B9285E]
    assert [int(x) for x in port.pcg64(42, 2)] == [0x287472E87FF5705A, 0xBBD190B04ED0B545]
    x = int(port.pcg64(2026, 1)[0])
    assert math.isclose((x >> 11) * 2.0 ** -53, 0.17980729564626807, rel_tol=1e-15)


def test_pcg64_and_gaussian_fixture(port):
    g = load_golden("pcg64")
    assert np.array_equal(port.pcg64(0, 64), g["s0"])
    assert np.array_equal(port.pcg64(42, 64), g["s42"])
    assert np.array_equal(port.pcg64(2026, 64), g["s2026"])
    assert np.array_equal(port.gaussian(33, 5, 0), g["gauss_0_33x5"])
    assert np.array_equal(port.gaussian(40, 8, 0 ^ 0x9E3779B97F4A7C15), g["gauss_sketch"])


def test_converged_count_prefix_rule(port):
    """tests/test_eigensolvers.cpp:180-199."""
    n = 10
    X = np.zeros((n, 3), order="F")
    R = np.zeros((n, 3), order="F")
    for j in range(3):
        X[j, j] = 1.0
    theta = [1.0, 2.0, 3.0]
    R[0, 0], R[0, 1], R[0, 2] = 1e-7, 1e-3, 1e-9
    assert port.converged_count(10.0, X, theta, R, 1e-6) == 1
    R[0, 1] = 1e-7
    assert port.converged_count(10.0, X, theta, R, 1e-6) == 3
    R[0, 0] = 1.0
    assert port.converged_count(10.0, X, theta, R, 1e-6) == 0


def lap_eigs(*ns):
    """analytic Dirichlet Laplacian spectrum (generators.cpp:32-46 in d dims)."""
    ev = np.zeros(1)
    for N in ns:
        s = 4 * np.sin(np.arange(1, N + 1) * np.pi / (2 * (N + 1))) ** 2
        ev = (ev[:, None] + s[None, :]).ravel()
    return np.sort(ev)


def test_oracle_recovers_analytic_spectrum(port):
    r = port.solve(Problem.lap3d(8), "mplobpcg-schol", k=4, tol=1e-10, maxit=500)
    assert r.status == 0 and r.converged
    assert np.abs(r.theta - lap_eigs(8, 8, 8)[:4]).max() / r.theta[0] < 1e-10
    r = port.solve(Problem.lap2d(12, 9), "dlobpcg-dchol", k=5, tol=1e-11, maxit=800)
    assert r.converged
    assert np.abs(r.theta - lap_eigs(12, 9)[:5]).max() / r.theta[0] < 1e-10


def test_small_eig_against_numpy(port):
    rng = np.random.default_rng(0)
    M = rng.standard_normal((40, 40))
    M = np.asfortranarray(M + M.T)
    st, v, V = port.small_herm_eig(M)
    assert st == 0
    assert np.abs(v - np.linalg.eigvalsh(M)).max() < 1e-12
    assert np.linalg.norm(M @ V - V * v) < 1e-11
    assert np.linalg.norm(V.T @ V - np.eye(40)) < 1e-12


@pytest.mark.parametrize("kappa", [1e1, 1e4, 1e7])
def test_mixed_qr_gate(port, kappa):
    """acceptance criterion 6 (acceptance.cpp:367-387): orthogonality <= 100*200*u_h."""
    rng = np.random.default_rng(1)
    n, m = 400, 12
    Q1, _ = np.linalg.qr(rng.standard_normal((n, m)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    A = np.asfortranarray((Q1 * kappa ** (-np.arange(m) / (m - 1))) @ Q2)
    st, Q, R = port.mixed_qr(A)
    assert st == 0
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) <= 100 * 200 * 2.0 ** -53
    assert np.all(np.diag(R) > 0)


# ---------------------------------------------------- restatement vs reference
CASES = [
    (Problem.lap3d(8), "dlobpcg-dchol", dict(k=4, tol=1e-10, maxit=500)),
    (Problem.lap3d(8), "dlobpcg-schol", dict(k=4, tol=1e-10, maxit=500)),
    (Problem.lap3d(8), "mplobpcg-schol", dict(k=4, tol=1e-10, maxit=500)),
    (Problem.lap3d(8), "pinvit", dict(k=4, tol=1e-10, maxit=5000)),
    (Problem.lap2d(9, 8), "mplobpcg-schol", dict(k=3, block=5, tol=1e-11, maxit=600, seed=42)),
    (Problem.lap3d(6, 5, 4), "dlobpcg-dchol", dict(k=6, tol=1e-10, maxit=600, seed=3)),
    (Problem.dense_matrix(spd_dense(80, 1e5, 41)[0]), "mplobpcg-schol",
     dict(k=3, block=5, tol=1e-11, maxit=800, seed=13)),
    (Problem.dense_matrix(spd_dense(80, 1e5, 41)[0]), "dlobpcg-dchol",
     dict(k=3, block=5, tol=1e-11, maxit=800, seed=13)),
]


@pytest.mark.parametrize("prob,variant,kw", CASES)
def test_port_matches_reference_bitwise(port, ref, prob, variant, kw):
    a = port.solve(prob, variant, **kw)
    b = ref.solve(prob, variant, **kw)
    assert a.status == b.status == 0
    assert (a.iters_lower, a.iters_working, a.converged) == (b.iters_lower, b.iters_working, b.converged)
    assert np.array_equal(a.theta, b.theta)
    assert np.array_equal(a.resid, b.resid)
    assert a.a_norm_est == b.a_norm_est
    assert np.array_equal(a.hist_ritz, b.hist_ritz)
    assert np.array_equal(a.hist_nc, b.hist_nc)


def test_port_kernels_match_reference(port, ref):
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.standard_normal((300, 9)))
    for name in ("householder_qr", "mixed_qr", "cholesky_qr"):
        sa, Qa, Ra = getattr(port, name)(A)
        sb, Qb, Rb = getattr(ref, name)(A)
        assert sa == sb == 0
        assert np.array_equal(Qa, Qb) and np.array_equal(Ra, Rb), name
    M = np.asfortranarray(A.T @ A)
    assert all(np.array_equal(x, y) for x, y in zip(port.small_herm_eig(M)[1:], ref.small_herm_eig(M)[1:]))
    S, _ = np.linalg.qr(rng.standard_normal((30, 12)))
    _, _, Cm = ref.small_herm_eig(np.asfortranarray(rng.standard_normal((12, 12)) + np.eye(12) * 3))
    for x, y in zip(port.hl_update(S, Cm, 4), ref.hl_update(S, Cm, 4)):
        assert np.array_equal(np.asarray(x), np.asarray(y))
    B, _ = np.linalg.qr(rng.standard_normal((300, 10)))
    assert np.array_equal(port.project_out(B, A, 2), ref.project_out(B, A, 2))
    D = A.copy()
    D[:, 3] = D[:, 1]
    assert np.array_equal(port.ortho_dropping(D, 1e-8), ref.ortho_dropping(D, 1e-8))
    X = np.asfortranarray(rng.standard_normal((8 * 7 * 6, 4)))
    assert np.array_equal(port.apply_op(Problem.lap3d(8, 7, 6), X), ref.apply_op(Problem.lap3d(8, 7, 6), X))


# ---------------------------------------------------- restatement vs fixtures
@pytest.mark.parametrize("name,prob", [
    ("lap3d8-dlobpcg-dchol", Problem.lap3d(8)),
    ("lap3d8-mplobpcg-schol", Problem.lap3d(8)),
    ("lap3d8-pinvit", Problem.lap3d(8)),
    ("lap2d50-mplobpcg-schol", Problem.lap2d(50)),
    ("dense256-mplobpcg-schol", None),
])
def test_port_matches_golden(port, name, prob):
    g = load_golden(name)
    if prob is None:
        prob = Problem.dense_matrix(spd_dense(256, 1e3, 5)[0])
    r = port.solve(prob, str(g["variant"]), **eval(str(g["kw"])))
    assert (r.iters_lower, r.iters_working) == (int(g["iters_lower"]), int(g["iters_working"]))
    assert np.array_equal(r.theta, g["theta"])
    assert np.array_equal(r.hist_resid, g["hist_resid"])
