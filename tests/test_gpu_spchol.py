"""Sparse Cholesky preconditioner on the device.

The reference's own preconditioner for sparse systems through its stock driver
solve(CsrMatrix, cfg) (drivers.hpp:183-210): RCM-permuted system, up-looking
factor (fp64 for DLOBPCG-dchol, fp32 of to_lower(A) otherwise, with
retry_sparse's shifted retry), eigenvectors unpermuted.  Golden fixtures:
tests/golden/make_golden.py (splap*, sprand*), produced by the reference.
"""
import numpy as np
import pytest

from conftest import load_golden
from problems import lap_csr, random_spd_csr
from test_gpu_solver import check_parity

pytestmark = pytest.mark.gpu

MATRICES = {
    "splap3d16": lambda: lap_csr(16, 16, 16),
    "splap2d50": lambda: lap_csr(50, 50),
    "sprand2000": lambda: random_spd_csr(2000, 3, 11),
    "splap3d8indef": lambda: lap_csr(8, 8, 8, shift=0.3618452752845494),
}
CASES = ["splap3d16-dlobpcg-dchol", "splap3d16-dlobpcg-schol", "splap3d16-mplobpcg-schol",
         "splap3d16-pinvit", "splap2d50-mplobpcg-schol", "sprand2000-mplobpcg-schol"]


def _solve(mp, name):
    g = load_golden(name)
    kw = eval(str(g["kw"]))  # dict literal written by make_golden.py
    kw.pop("native", None)
    cfg = mp.SolverConfig(variant=str(g["variant"]), **kw)
    rp, ci, v = MATRICES[name.split("-")[0]]()
    return g, cfg, (rp, ci, v), mp.solve_csr(rp, ci, v, cfg)


def _band(name):
    """+-2, widened to 2 x the reference's own spread under +-1 binary32-ulp
    perturbations of diag(A) where measured (tests/golden/make_sparse_sensitivity.py;
    the band policy of DESIGN.md §4.2).  sprand2000 mixed: the reference itself
    moves by up to 6 iterations (116..127 around 121): a clustered spectrum."""
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                     "sensitivity_sparse.json")
    spread = json.load(open(p)).get(name, {}).get("spread", 0) if os.path.exists(p) else 0
    return max(2, 2 * spread)


@pytest.mark.parametrize("name", CASES)
def test_sparse_cholesky_solve_parity(gpu, name):
    """theta within 1e-10, residual contract, iterations within +-2 of the reference
    (or the reference's own measured rounding spread, _band)."""
    g, cfg, _, r = _solve(gpu, name)
    assert r.precond_shift == 0.0
    check_parity(g, cfg, r, name, iter_slack=_band(name))


def test_sparse_cholesky_eigenvectors_unpermuted(gpu):
    """X comes back in the original row order: ||A x - theta x|| small on the
    ORIGINAL matrix (drivers.hpp:209 unpermute_rows)."""
    g, cfg, (rp, ci, v), r = _solve(gpu, "splap3d16-mplobpcg-schol")
    import scipy.sparse as sp
    n = rp.size - 1
    A = sp.csr_matrix((v, ci, rp), shape=(n, n))
    X = np.asarray(r.X)
    X = X.T if X.shape[0] != n else X
    R = A @ X - X * r.theta
    thr = cfg.tol * (r.a_norm_estimate + np.abs(r.theta))
    assert np.all(np.linalg.norm(R, axis=0) <= 10 * thr)


def test_sparse_cholesky_retry_shift(gpu):
    """lambda_min = -1e-6: the fp32 factor breaks down, the factor is rebuilt from
    A + 10 u_l ||A||_est I; the shift is the reference's (kShiftSeed sketch)."""
    g, cfg, _, r = _solve(gpu, "splap3d8indef-dlobpcg-schol")
    ref_shift = float(g["precond_shift"])
    assert ref_shift > 0
    assert abs(r.precond_shift - ref_shift) <= 1e-12 * ref_shift
    assert not r.converged and not bool(g["converged"])
    assert r.iterations_working == int(g["iters_working"])


def test_sparse_cholesky_apply_matches_solve(gpu):
    """apply(R) = A^-1 R: fp64 factor to 1e-12 (RCM, identity and user orderings
    agree), the fp32 sandwich and apply_lower to the binary32 accuracy."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    import torch
    mp = gpu
    rp, ci, v = random_spd_csr(2000, 3, 11)
    n = rp.size - 1
    A = mp.csr_matrix(rp, ci, v)
    As = sp.csr_matrix((v, ci, rp), shape=(n, n)).tocsc()
    rng = np.random.default_rng(0)
    Rh = rng.standard_normal((n, 5))
    ref = sla.spsolve(As, Rh)
    R = torch.tensor(Rh.T.copy(), device="cuda")
    for perm in ("rcm", None, rng.permutation(n)):
        T = mp.sparse_cholesky(A, mp.WORKING, perm=perm)
        W = T.apply(R, precision=mp.WORKING).cpu().numpy().T
        assert np.abs(W - ref).max() <= 1e-12 * np.abs(ref).max(), perm
        assert T.factor_nnz >= (ci.size + n) // 2
    Tl = mp.sparse_cholesky(A, mp.LOWER)
    W = Tl.apply(R, precision=mp.WORKING).cpu().numpy().T
    assert np.abs(W - ref).max() / np.abs(ref).max() <= 1e-5
    assert np.all(W.astype(np.float32).astype(np.float64) == W)  # to_working of fp32
    Wl = Tl.apply(R.float(), precision=mp.LOWER).double().cpu().numpy().T
    assert np.array_equal(Wl, W)
    # in place (W aliases R) gives the same result
    R2 = R.clone()
    T = mp.sparse_cholesky(A, mp.WORKING)
    T.apply(R2, Y=R2, precision=mp.WORKING)
    assert np.abs(R2.cpu().numpy().T - ref).max() <= 1e-12 * np.abs(ref).max()


def test_sparse_cholesky_errors(gpu):
    mp = gpu
    with pytest.raises(mp.ConfigError):
        mp.sparse_cholesky(mp.laplace3d(4), mp.WORKING)
    rp, ci, v = lap_csr(4, 4, 4, shift=7.0)  # diagonal -1: not positive definite
    with pytest.raises(mp.NotPositiveDefinite) as ei:
        mp.sparse_cholesky(mp.csr_matrix(rp, ci, v), mp.WORKING, perm=None)
    assert ei.value.index == 0
    rp, ci, v = lap_csr(4, 4, 4)
    with pytest.raises(mp.DimensionMismatch):
        mp.sparse_cholesky(mp.csr_matrix(rp, ci, v), mp.WORKING, perm=np.zeros(64, np.int64))
    import torch
    T = mp.sparse_cholesky(mp.csr_matrix(rp, ci, v), mp.WORKING)
    with pytest.raises(mp.ConfigError):
        T.apply(torch.ones((1, 64), dtype=torch.float32, device="cuda"), precision=mp.LOWER)


@pytest.mark.parametrize("prec", ["working", "lower"])
def test_parallel_host_factor_is_bitwise_sequential(gpu, prec):
    """The up-looking factor with rows in flight on host threads (spchol_host.cpp)
    forms every entry by the same operations in the same order as one thread:
    the preconditioner applies bitwise identically for any thread count."""
    import torch
    mp = gpu
    rp, ci, v = lap_csr(20, 22, 18)
    n = len(rp) - 1
    A = mp.csr_matrix(rp, ci, v)
    p = mp.WORKING if prec == "working" else mp.LOWER
    dt = np.float64 if prec == "working" else np.float32
    X = mp.to_device(np.asfortranarray(np.random.default_rng(9).standard_normal((n, 5)).astype(dt)))
    ctx = A.ctx
    outs = []
    try:
        for th in (1, 3, 8):
            assert ctx.lib.mpeig_set_process_option(b"spchol_threads", th) == 0
            T = mp.sparse_cholesky(A, p)
            outs.append((T.factor_nnz, mp.to_host(T.apply(X, precision=p))))
            torch.cuda.synchronize()
    finally:
        ctx.lib.mpeig_set_process_option(b"spchol_threads", 0)
    for nnz, Y in outs[1:]:
        assert nnz == outs[0][0]
        assert np.array_equal(Y, outs[0][1])


def test_parallel_host_factor_reports_first_failing_row(gpu):
    """An indefinite system: every thread count reports the sequential algorithm's
    first nonpositive pivot (the lowest failing row)."""
    mp = gpu
    rp, ci, v = lap_csr(18, 17, 16, shift=0.5)  # lambda_min < 0.5: indefinite
    A = mp.csr_matrix(rp, ci, v)
    ctx = A.ctx
    idx = []
    try:
        for th in (1, 6):
            assert ctx.lib.mpeig_set_process_option(b"spchol_threads", th) == 0
            with pytest.raises(mp.NotPositiveDefinite) as e:
                mp.sparse_cholesky(A, mp.WORKING, perm=None)
            idx.append(e.value.index)
    finally:
        ctx.lib.mpeig_set_process_option(b"spchol_threads", 0)
    assert idx[0] == idx[1] and idx[0] >= 0
