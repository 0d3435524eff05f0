"""Harness-defined test matrices shared by make_golden.py and the tests."""
import numpy as np


def spd_dense(n: int, kappa: float, seed: int):
    """Dense SPD matrix with a prescribed log-spaced spectrum in [1, kappa].

    Harness-defined (cfg3 family): A = Q diag(lam) Q^T with Q a
    product of 3 seeded Householder reflectors (the recipe of the reference's
    oracles.hpp:234-279), built with numpy.  The same bytes are fed to the
    reference, the C restatement and the GPU path.
    """
    rng = np.random.default_rng(seed)
    lam = np.sort(np.exp(np.log(kappa) * rng.random(n)))
    lam[0], lam[-1] = 1.0, kappa
    Q = np.eye(n)
    for _ in range(3):
        v = rng.standard_normal(n)
        Q = Q - np.outer(Q @ v, v) * (2.0 / (v @ v))
    A = (Q * lam) @ Q.T
    A = 0.5 * (A + A.T)
    return np.asfortranarray(A), lam
