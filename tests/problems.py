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


def lap_csr(nx: int, ny: int, nz: int = 1, shift: float = 0.0):
    """7-pt (nz > 1) / 5-pt (nz = 1) Dirichlet Laplacian as CSR, row = x + nx (y + ny z),
    columns ascending, diagonal 6 (4) - shift, off-diagonals -1 (the reference's
    gen_laplace2d, generators.cpp:13-30, and its 3-D analogue)."""
    import numpy as np
    n = nx * ny * nz
    d = (6.0 if nz > 1 else 4.0) - shift
    rp, ci, v = [0], [], []
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                i = x + nx * (y + ny * z)
                ent = []
                if z > 0:
                    ent.append((i - nx * ny, -1.0))
                if y > 0:
                    ent.append((i - nx, -1.0))
                if x > 0:
                    ent.append((i - 1, -1.0))
                ent.append((i, d))
                if x < nx - 1:
                    ent.append((i + 1, -1.0))
                if y < ny - 1:
                    ent.append((i + nx, -1.0))
                if z < nz - 1:
                    ent.append((i + nx * ny, -1.0))
                for c, val in ent:
                    ci.append(c)
                    v.append(val)
                rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int64), np.array(v)


def random_spd_csr(n: int, per_row: int, seed: int):
    """Random symmetric sparse pattern (per_row off-diagonals per row before
    symmetrisation), diagonally dominant values: an RCM / sparse-Cholesky test case."""
    import numpy as np
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n), per_row)
    cols = rng.integers(0, n, n * per_row)
    keep = rows != cols
    r = np.concatenate([rows[keep], cols[keep]])
    c = np.concatenate([cols[keep], rows[keep]])
    val = -rng.random(keep.sum())
    val = np.concatenate([val, val])
    A = {}
    for a, b, x in zip(r.tolist(), c.tolist(), val.tolist()):
        A[(a, b)] = A.get((a, b), 0.0) + x
    off = np.zeros(n)
    for (a, b), x in A.items():
        off[a] += abs(x)
    for i in range(n):
        A[(i, i)] = off[i] + 1.0
    keys = sorted(A)
    rp = np.zeros(n + 1, np.int64)
    for a, _ in keys:
        rp[a + 1] += 1
    return (np.cumsum(rp), np.array([b for _, b in keys], np.int64),
            np.array([A[k] for k in keys]))


def perturb_x0(X0, p: int, ulp: str = "f64"):
    """Start block with rounding-level noise: every entry of X0 moved by -1, 0 or
    +1 ulp, chosen by a seeded generator (p = 0: X0 unchanged).  ulp = "f64":
    one binary64 ulp (np.nextafter) -- the working-precision modes; "f32": one
    binary32 ulp of the entry -- the mixed mode, whose fp32 stage 1 would round
    a binary64-ulp nudge away in to_lower.  Fed to the reference (oracle x0
    override) and to the device alike; the spread of the reference's own
    iteration counts over p = 1..16 is the iteration-parity envelope
    (tests/golden/make_envelope.py)."""
    X0 = np.asfortranarray(X0, dtype=np.float64)
    if p == 0:
        return X0.copy(order="F")
    d = np.random.default_rng(0x5EED0000 + p).integers(-1, 2, size=X0.shape)
    if ulp == "f32":
        step = np.spacing(np.abs(X0).astype(np.float32)).astype(np.float64)
        return np.asfortranarray(X0 + d * step)
    up, dn = np.nextafter(X0, np.inf), np.nextafter(X0, -np.inf)
    return np.asfortranarray(np.where(d > 0, up, np.where(d < 0, dn, X0)))


def envelope_ulp(variant: str) -> str:
    """Perturbation scale of the envelope for a variant (perturb_x0)."""
    return "f32" if variant == "mplobpcg-schol" else "f64"
