"""Rounding-error bound analysis (analysis.hpp / analysis.cpp:8-84 of the reference) and
the per-run BoundReport the reference's bench CLI emits under --bounds
(tools/bench_main.cpp:116-171), for the run reports of run_record.py.

Host-side reporting: the scalar bounds are closed-form; the two measured quantities
(gamma_precond = ||I - A^1/2 T_E A^1/2||_2 and ||T_E|| ||A||) densify the ACTUAL device
preconditioner by applying it to the identity / to A^1/2 through the library, so every
rounding of the device solve chain is included, as in the reference.  Like the
reference's CLI this is for small operators (n <= 200: dense O(n^3) host algebra).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .api import MpeigError

U_WORKING = 2.0 ** -53  # kUnitRoundoffWorking (binary64)
U_LOWER = 2.0 ** -24    # kUnitRoundoffLower (binary32)


class AssumptionViolated(MpeigError, ValueError):
    """A hypothesis of the bound does not hold (errors.hpp)."""


class BoundVacuous(MpeigError, ValueError):
    """The bound evaluates to >= 1 and certifies nothing."""


class OutOfInterval(MpeigError, ValueError):
    """rho outside (lambda1, lambda2)."""


class GammaTooLarge(MpeigError, ValueError):
    """gamma >= 1: no contraction."""


class DenominatorNonpositive(MpeigError, ArithmeticError):
    """1 - gamma - gamma_2 ||T|| ||A|| <= 0 in the accuracy floor."""


def gamma_n(n: int, u: float) -> float:
    """gamma_n = n u / (1 - n u) (analysis.cpp:8-13)."""
    if not u >= 0:
        raise AssumptionViolated("gamma_n: negative unit roundoff")
    nu = float(n) * u
    if nu >= 1:
        raise AssumptionViolated("gamma_n: n*u >= 1")
    return nu / (1.0 - nu)


def epsilon_A(n: int, u_h: float) -> float:
    """Backward error of a rounded Hermitian apply, sqrt(n) gamma_n (:15-17)."""
    return math.sqrt(float(n)) * gamma_n(n, u_h)


def epsilon_r(n: int, u_h: float, eps_A: float) -> float:
    """Normwise error of a computed residual (:19-25)."""
    nd = float(n)
    if 2.0 * nd * u_h >= 1:
        raise AssumptionViolated("epsilon_r: 2*n*u_h >= 1")
    g = gamma_n(n, u_h)
    num = (g + eps_A + g * eps_A + (nd + 1.0) * u_h) * (1.0 + u_h)
    return num / (1.0 - 2.0 * nd * u_h) + eps_A + u_h


def epsilon_T(n: int, kappa: float, u_l: float) -> float:
    """Quality of a Cholesky solve at unit roundoff u_l: 4n(3n+1) kappa u_l (:27-35)."""
    if not kappa >= 1:
        raise AssumptionViolated("epsilon_T: kappa < 1")
    nd = float(n)
    v = 4.0 * nd * (3.0 * nd + 1.0) * kappa * u_l
    if v >= 1:
        raise BoundVacuous(f"epsilon_T: 4n(3n+1) kappa u_l = {v} >= 1")
    return v


def gamma_precond_bound(n: int, kappa: float, u_l: float) -> float:
    """||I - A^1/2 T A^1/2|| <= eps_T / (1 - eps_T) (:37-40)."""
    e = epsilon_T(n, kappa, u_l)
    return e / (1.0 - e)


def beta(rho: float, lambda1: float, lambda2: float, lambdan: float) -> float:
    """max{sqrt(l1 ln)/(rho-l1), sqrt(l2 ln)/(l2-rho)} for rho in (l1, l2) (:42-50)."""
    if not (0 < lambda1 < lambda2 <= lambdan):
        raise AssumptionViolated("beta: need 0 < lambda1 < lambda2 <= lambdan")
    if not (lambda1 < rho < lambda2):
        raise OutOfInterval("beta: rho outside (lambda1, lambda2)")
    b1 = math.sqrt(lambda1 * lambdan) / (rho - lambda1)
    b2 = math.sqrt(lambda2 * lambdan) / (lambda2 - rho)
    return b1 if b1 > b2 else b2


def gamma_total(gamma_precond: float, norm_te_norm_a: float, beta_val: float, n: int,
                u_h: float, eps_r: float) -> float:
    """Effective contraction of one preconditioned step (:52-61)."""
    if float(n) * u_h >= 1:
        raise AssumptionViolated("gamma_total: n*u_h >= 1")
    if not (gamma_precond >= 0 and norm_te_norm_a >= 0 and beta_val >= 0 and eps_r >= 0):
        raise AssumptionViolated("gamma_total: negative input")
    g2 = gamma_n(2, u_h)
    return gamma_precond + g2 * norm_te_norm_a + beta_val * (u_h + (1.0 + g2) * eps_r * norm_te_norm_a)


def rate_bound(gamma: float, lambda1: float, lambda2: float) -> float:
    """One-step bound (gamma + (1 - gamma) l1/l2)^2 (:63-70)."""
    if not (0 < lambda1 < lambda2):
        raise AssumptionViolated("rate_bound: need 0 < lambda1 < lambda2")
    if not gamma >= 0:
        raise AssumptionViolated("rate_bound: gamma < 0")
    if gamma >= 1:
        raise GammaTooLarge("rate_bound: gamma >= 1")
    base = gamma + (1.0 - gamma) * lambda1 / lambda2
    return base * base


def accuracy_floor(gamma_precond: float, norm_te_norm_a: float, n: int, u_h: float, eps_r: float,
                   lambda1: float, lambdan: float) -> float:
    """Smallest eigenvalue error the finite-precision iteration certifies (:72-84)."""
    if not (0 < lambda1 <= lambdan):
        raise AssumptionViolated("accuracy_floor: need 0 < lambda1 <= lambdan")
    if float(n) * u_h >= 1:
        raise AssumptionViolated("accuracy_floor: n*u_h >= 1")
    g2 = gamma_n(2, u_h)
    denom = 1.0 - gamma_precond - g2 * norm_te_norm_a
    if not denom > 0:
        raise DenominatorNonpositive("accuracy_floor: 1 - gamma - g2||T||||A|| <= 0")
    num = u_h + (1.0 + g2) * eps_r * norm_te_norm_a
    return math.sqrt(lambda1 * lambdan) * num / denom


# ----------------------------------------------------------- measured quantities


def operator_norm_2(M) -> float:
    """||M||_2 from the largest eigenvalue of M^T M (analysis.hpp:48-56)."""
    M = np.asarray(M, dtype=np.float64)
    if M.size == 0:
        return 0.0
    lmax = float(np.linalg.eigvalsh(M.T @ M)[-1])
    return math.sqrt(lmax if lmax > 0 else 0.0)


def _apply_dense(T, B):
    """T (a device preconditioner Operator) applied to the columns of host B."""
    from .api import WORKING, to_device, to_host
    return to_host(T.apply(to_device(np.asfortranarray(B, dtype=np.float64)), precision=WORKING))


def densify_preconditioner(T) -> np.ndarray:
    """T_E = the device preconditioner applied to I (analysis.hpp:58-62)."""
    return _apply_dense(T, np.eye(T.n))


def measure_gamma_precond(A, T) -> float:
    """gamma = ||I - A^1/2 T_E A^1/2||_2 through the actual device apply (:64-92)."""
    from .api import DimensionMismatch, NotPositiveDefinite
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise DimensionMismatch("measure_gamma_precond: A not square", -1)
    if A.shape[0] != T.n:
        raise DimensionMismatch("measure_gamma_precond: preconditioner size differs", -1)
    lam, V = np.linalg.eigh(A)
    if lam.size and not lam[0] > 0:
        raise NotPositiveDefinite("measure_gamma_precond: A is not positive definite", 0)
    Ahalf = (V * np.sqrt(lam)) @ V.T
    G = np.eye(A.shape[0]) - Ahalf @ _apply_dense(T, Ahalf)
    return operator_norm_2(G)


@dataclass
class BoundReport:
    """Everything the reference's CLI reports under --bounds (analysis.hpp:95-109)."""
    n: int = 0
    kappa: float = 0.0
    eps_A: float = 0.0
    eps_r: float = 0.0
    eps_T: float = 0.0
    eps_T_vacuous: bool = False
    gamma_precond_meas: float = 0.0
    norm_te_norm_a: float = 0.0
    beta_mid: float = 0.0
    gamma_total_mid: float = 0.0
    rate_mid: float = 0.0
    floor: float = 0.0


def bounds_for(A, variant: str, ctx=None) -> BoundReport:
    """bounds_for (tools/bench_main.cpp:116-171) on a dense copy of A (n <= 200): the
    spectrum from a dense eigensolve, the run's preconditioner (dense Cholesky built in
    the working precision for DLOBPCG-dchol, else the lower) measured through the
    device apply, beta / gamma / rate at the midpoint rho = (l1 + l2) / 2."""
    from .api import WORKING, LOWER, default_context, dense_cholesky, dense_matrix
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    if n > 200:
        raise AssumptionViolated("--bounds is limited to n <= 200")
    b = BoundReport(n=n)
    lam = np.linalg.eigvalsh(A)
    l1, ln = float(lam[0]), float(lam[-1])
    l2 = float(lam[1] if lam.size > 1 else lam[0])
    b.kappa = ln / l1
    b.eps_A = epsilon_A(n, U_WORKING)
    b.eps_r = epsilon_r(n, U_WORKING, b.eps_A)
    b.eps_T = 4.0 * n * (3.0 * n + 1.0) * b.kappa * U_LOWER
    b.eps_T_vacuous = b.eps_T >= 1.0
    ctx = ctx or default_context()
    Aop = dense_matrix(A, ctx=ctx)
    T = dense_cholesky(Aop, WORKING if variant == "dlobpcg-dchol" else LOWER)
    b.gamma_precond_meas = measure_gamma_precond(A, T)
    b.norm_te_norm_a = operator_norm_2(densify_preconditioner(T)) * operator_norm_2(A)
    rho = 0.5 * (l1 + l2)
    if l1 < rho < l2 <= ln:
        b.beta_mid = beta(rho, l1, l2, ln)
        b.gamma_total_mid = gamma_total(b.gamma_precond_meas, b.norm_te_norm_a, b.beta_mid, n,
                                        U_WORKING, b.eps_r)
        b.rate_mid = (rate_bound(b.gamma_total_mid, l1, l2) if b.gamma_total_mid < 1.0
                      else math.inf)
    else:  # degenerate leading eigenvalue: no interval to certify
        b.beta_mid = b.gamma_total_mid = b.rate_mid = math.inf
    try:
        b.floor = accuracy_floor(b.gamma_precond_meas, b.norm_te_norm_a, n, U_WORKING, b.eps_r,
                                 l1, ln)
    except DenominatorNonpositive:
        b.floor = math.inf
    return b
