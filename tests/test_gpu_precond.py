"""Dense Cholesky preconditioner on the device.

The reference's own preconditioner for dense systems, Preconditioner<T>::build
(DenseMatrix, prec) (precond.hpp:33-50): an fp64 factor for DLOBPCG-dchol, an
fp32 factor of to_lower(A) otherwise, with retry_dense's shifted retry
(:140-146).  Golden fixtures: the reference's stock solve(DenseMatrix, cfg)
(drivers.hpp:158-181) run by tests/golden/make_golden.py (dense256chol-*).
"""
import numpy as np
import pytest

from conftest import load_golden
from problems import spd_dense
from test_gpu_solver import check_parity

pytestmark = pytest.mark.gpu

CASES = ["dense256chol-dlobpcg-dchol", "dense256chol-dlobpcg-schol",
         "dense256chol-mplobpcg-schol", "dense256chol-pinvit"]


def _solve(mp, name, kappa=1e3):
    g = load_golden(name)
    kw = eval(str(g["kw"]))  # dict literal written by make_golden.py
    kw.pop("native", None)
    variant = str(g["variant"])
    A = mp.dense_matrix(spd_dense(256, kappa, 5)[0])
    T = mp.dense_cholesky(A, mp.build_precision_for(variant))
    cfg = mp.SolverConfig(variant=variant, **kw)
    return g, cfg, T, mp.solve(A, cfg, T=T)


@pytest.mark.parametrize("name", CASES)
def test_dense_cholesky_solve_parity(gpu, name):
    """theta within 1e-10, residual contract, iterations within +-2 of the reference."""
    g, cfg, T, r = _solve(gpu, name)
    assert T.shift == 0.0
    check_parity(g, cfg, r, name, iter_slack=2)


def test_dense_cholesky_retry_shift(gpu):
    """kappa = 1e10: to_lower(A) is not positive definite in fp32, so the factor is
    rebuilt from A + 10 u_l ||A||_est I; the shift is the reference's (same sketch
    seed kShiftSeed, precond.hpp:161) to the Frobenius-sum rounding."""
    g, cfg, T, r = _solve(gpu, "dense256chol-k1e10-dlobpcg-schol", kappa=1e10)
    ref_shift = float(g["precond_shift"])
    assert ref_shift > 0
    assert abs(T.shift - ref_shift) <= 1e-12 * ref_shift
    assert not r.converged and not bool(g["converged"])
    assert r.iterations_working == int(g["iters_working"])


def test_dense_cholesky_apply_matches_solve(gpu):
    """apply(R) = A^-1 R: fp64 factor to 1e-12, the fp32 sandwich / apply_lower to
    the binary32 solve accuracy (kappa = 1e3)."""
    import torch
    mp = gpu
    Ah = spd_dense(256, 1e3, 5)[0]
    A = mp.dense_matrix(Ah)
    rng = np.random.default_rng(0)
    R = rng.standard_normal((256, 7))
    ref = np.linalg.solve(Ah, R)
    Rt = torch.tensor(R.T.copy(), device="cuda")  # (ncols, ld) = column-major n x c
    Tw = mp.dense_cholesky(A, mp.WORKING)
    W = Tw.apply(Rt, precision=mp.WORKING).cpu().numpy().T
    assert np.abs(W - ref).max() <= 1e-12 * np.abs(ref).max()
    Tl = mp.dense_cholesky(A, mp.LOWER)
    W = Tl.apply(Rt, precision=mp.WORKING).cpu().numpy().T
    err = np.abs(W - ref).max() / np.abs(ref).max()
    assert 0 < err <= 1e3 * 2.0 ** -24 * 10
    # apply returns exact fp32 values widened (to_working of an fp32 block)
    assert np.all(W.astype(np.float32).astype(np.float64) == W)
    Wl = Tl.apply(Rt.float(), precision=mp.LOWER).cpu().numpy().T
    assert np.abs(Wl - ref).max() / np.abs(ref).max() <= 1e3 * 2.0 ** -24 * 10
    # the working-precision sandwich is to_working(apply_lower(to_lower(R)))
    Wl2 = Tl.apply(Rt.float(), precision=mp.LOWER).double().cpu().numpy().T
    assert np.array_equal(Wl2, W)


def test_dense_cholesky_errors(gpu):
    mp = gpu
    # not an explicit dense matrix (precond.hpp builds from DenseMatrix / CsrMatrix)
    with pytest.raises(mp.ConfigError):
        mp.dense_cholesky(mp.laplace3d(4), mp.WORKING)
    # indefinite: NotPositiveDefinite with the failing pivot (dense_kernels.hpp:144-146);
    # no retry in working precision (precond.hpp:38-41)
    Ah = np.eye(16)
    Ah[5, 5] = -1.0
    with pytest.raises(mp.NotPositiveDefinite) as ei:
        mp.dense_cholesky(mp.dense_matrix(Ah), mp.WORKING)
    assert ei.value.index == 5
    # apply_lower of a working-precision factor (precond.hpp:103-105)
    import torch
    T = mp.dense_cholesky(mp.dense_matrix(np.eye(16) * 2.0), mp.WORKING)
    with pytest.raises(mp.ConfigError):
        T.apply(torch.ones((1, 16), dtype=torch.float32, device="cuda"), precision=mp.LOWER)


@pytest.mark.parametrize("name", ["dense2048chol-dlobpcg-dchol", "dense2048chol-mplobpcg-schol"])
def test_dense_cholesky_m96(gpu, name):
    """cfg3's block (k = 64, m = 96, s = 288) with the reference's dense Cholesky
    preconditioner on a 2048 x 2048 SPD matrix: the stock solve(DenseMatrix)."""
    mp = gpu
    g = load_golden(name)
    kw = eval(str(g["kw"]))
    kw.pop("native", None)
    variant = str(g["variant"])
    A = mp.dense_matrix(spd_dense(2048, 1e3, 9)[0])
    T = mp.dense_cholesky(A, mp.build_precision_for(variant))
    cfg = mp.SolverConfig(variant=variant, **kw)
    r = mp.solve(A, cfg, T=T)
    check_parity(g, cfg, r, name, iter_slack=2)


@pytest.mark.gpu
def test_bound_report_measured_through_device_preconditioner(gpu):
    """--bounds (bench_main.cpp:116-171, test_analysis.cpp:159-176): gamma measured by
    densifying the DEVICE dense-Cholesky preconditioner; the working build is
    essentially exact, the binary32 build inside Lemma 2's bound."""
    import paper_2302_12528_b200.analysis as an
    from problems import spd_dense
    n, kappa = 30, 100.0
    A, lam = spd_dense(n, kappa, 31)
    bw = an.bounds_for(A, "dlobpcg-dchol")
    bl = an.bounds_for(A, "mplobpcg-schol")
    assert abs(bw.kappa - lam[-1] / lam[0]) <= 1e-8 * bw.kappa
    assert bw.gamma_precond_meas < 1e4 * kappa * 2.0 ** -53
    assert bw.gamma_precond_meas < bl.gamma_precond_meas <= an.gamma_precond_bound(n, kappa, 2.0 ** -24)
    assert bl.norm_te_norm_a == pytest.approx(kappa, rel=1e-3)
    assert 0 < bl.rate_mid < 1 and 0 < bl.floor < 1e-10
    from paper_2302_12528_b200.run_record import RunRecord, run_record_csv
    rec = RunRecord("spd30", n, n * n, "mplobpcg-schol", 2, 3, 0, 1, 1, True, [1.0, 2.0], [0, 0],
                    bounds=bl)
    assert ",kappa," in run_record_csv([rec])
