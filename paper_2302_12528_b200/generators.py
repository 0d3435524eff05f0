"""Synthetic workload generators (harness-defined; the reference has none for
these families).  Pure numpy: importable without the CUDA library.

cfg5 (BASELINE.json configs[4]): a Kohn-Sham-like operator
H = -Laplacian_7pt + V on an nx x ny x nz Dirichlet grid, V a seeded sum of
Gaussian potential wells.  Its low spectrum is clustered: bound states of
wells with similar depth and width, the regime the paper's KS motivation
targets.
"""
from __future__ import annotations

import numpy as np


def ks_potential(nx: int, ny: int, nz: int, nwells: int = 12, seed: int = 0,
                 depth: tuple = (2.0, 4.0), width: tuple = (0.05, 0.10)) -> np.ndarray:
    """V on the grid, row = x + nx (y + ny z) (the 7-pt Laplacian's order).

    V(r) = max(0, D - sum_w d_w exp(-|r - c_w|^2 / (2 s_w^2))) with r =
    ((x+1)/(nx+1), (y+1)/(ny+1), (z+1)/(nz+1)) in the unit cube, well centres
    c_w uniform in [0.15, 0.85]^3, depths d_w uniform in `depth`, widths s_w
    uniform in `width`, and D = max_w d_w: the background sits at D, the
    deepest well reaches 0, so V >= 0 and H = -Laplacian + V is SPD with a
    low spectrum of well-bound states.  All draws come from numpy's PCG64
    stream for `seed`."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.15, 0.85, size=(nwells, 3))
    d = rng.uniform(depth[0], depth[1], size=nwells)
    s = rng.uniform(width[0], width[1], size=nwells)
    gx = (np.arange(nx) + 1.0) / (nx + 1)
    gy = (np.arange(ny) + 1.0) / (ny + 1)
    gz = (np.arange(nz) + 1.0) / (nz + 1)
    V = np.full((nz, ny, nx), float(d.max()))
    for w in range(nwells):
        ex = np.exp(-(gx - c[w, 0]) ** 2 / (2 * s[w] ** 2))
        ey = np.exp(-(gy - c[w, 1]) ** 2 / (2 * s[w] ** 2))
        ez = np.exp(-(gz - c[w, 2]) ** 2 / (2 * s[w] ** 2))
        V -= d[w] * ez[:, None, None] * ey[None, :, None] * ex[None, None, :]
    return np.maximum(V, 0.0).ravel()


def ks_diagonal(nx: int, ny: int, nz: int, seed: int = 0, **kw) -> np.ndarray:
    """The diagonal 6 + V_i of H = -Laplacian_7pt + V."""
    return 6.0 + ks_potential(nx, ny, nz, seed=seed, **kw)


def ks_csr(nx: int, ny: int, nz: int, seed: int = 0, **kw):
    """H as CSR (int64 row_ptr / col_idx, columns ascending per row): the same
    matrix the reference builds with CsrMatrix::from_triplets."""
    n = nx * ny * nz
    diag = ks_diagonal(nx, ny, nz, seed=seed, **kw)
    idx = np.arange(n).reshape(nz, ny, nx)
    rows, cols, vals = [], [], []
    for dz, dy, dx in ((-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0)):
        z0, z1 = max(0, -dz), nz - max(0, dz)
        y0, y1 = max(0, -dy), ny - max(0, dy)
        x0, x1 = max(0, -dx), nx - max(0, dx)
        r = idx[z0:z1, y0:y1, x0:x1].ravel()
        cc = idx[z0 + dz:z1 + dz, y0 + dy:y1 + dy, x0 + dx:x1 + dx].ravel()
        rows.append(r)
        cols.append(cc)
        vals.append(diag[r] if (dz, dy, dx) == (0, 0, 0) else np.full(r.size, -1.0))
    r, cc, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    o = np.lexsort((cc, r))
    r, cc, v = r[o], cc[o], v[o]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp), cc.astype(np.int64), v
