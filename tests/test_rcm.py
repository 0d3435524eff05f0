"""Reverse Cuthill-McKee ordering of the sparse Cholesky preconditioner.

mpeig_rcm_ordering (host code in libmpeig_b200.so) against the reference's
rcm_ordering_pattern (rcm.cpp:8-57) on fixtures the reference produced
(tests/golden/make_golden.py -> rcm.npz).  The ordering fixes the factor's
pattern, so it must be identical, not merely as good.  CPU-only.
"""
import numpy as np

from conftest import load_golden
from problems import lap_csr, random_spd_csr


def _cases():
    return {"lap3d8": lap_csr(8, 8, 8), "lap2d5x500": lap_csr(5, 500),
            "lap3d12x7x5": lap_csr(12, 7, 5), "rand2000": random_spd_csr(2000, 3, 11)}


def test_rcm_matches_reference():
    import paper_2302_12528_b200 as mp
    g = load_golden("rcm")
    for name, (rp, ci, _) in _cases().items():
        perm = mp.rcm_ordering(rp, ci)
        assert np.array_equal(perm, g[name]), name
        assert np.array_equal(np.sort(perm), np.arange(rp.size - 1))


def test_rcm_diagonal_and_components():
    """Isolated vertices and component order are unaffected (rcm.cpp:51-53): a
    diagonal matrix keeps the identity ordering; two disjoint paths stay apart."""
    import paper_2302_12528_b200 as mp
    n = 7
    rp, ci = np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64)
    assert np.array_equal(mp.rcm_ordering(rp, ci), np.arange(n))
    # path 0-1-2 and path 3-4 (symmetric pattern with diagonal)
    rows = {0: [0, 1], 1: [0, 1, 2], 2: [1, 2], 3: [3, 4], 4: [3, 4]}
    rp = np.cumsum([0] + [len(rows[i]) for i in range(5)]).astype(np.int64)
    ci = np.array(sum((rows[i] for i in range(5)), []), np.int64)
    perm = mp.rcm_ordering(rp, ci)
    assert sorted(perm[:3].tolist()) == [0, 1, 2] or sorted(perm[:2].tolist()) == [3, 4]
    assert sorted(perm.tolist()) == list(range(5))
