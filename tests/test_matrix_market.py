"""Matrix Market ingestion: read_matrix_market mirrors the
reference's read_matrix_market_real (matrix_market.cpp:128-157, 204-215) and
CsrMatrix::from_triplets (csr_matrix.hpp:31-58).  CPU-only."""
import numpy as np
import pytest

from problems import lap_csr


def _write(tmp_path, text, name="a.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_symmetric_mirrored_duplicates_accumulate(tmp_path):
    import paper_2302_12528_b200 as mp
    path = _write(tmp_path, "%%MatrixMarket matrix coordinate real symmetric\n"
                            "% a comment\n\n3 3 5\n1 1 4\n2 1 -1\n3 3 2.5\n2 2 4\n3 3 0.5\n")
    rp, ci, v = mp.read_matrix_market(path)
    A = np.zeros((3, 3))
    for i in range(3):
        for p in range(rp[i], rp[i + 1]):
            A[i, ci[p]] = v[p]
    assert np.array_equal(A, [[4, -1, 0], [-1, 4, 0], [0, 0, 3.0]])
    assert all(np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0) for i in range(3))


def test_roundtrip_laplacian_lower_triangle(tmp_path):
    import paper_2302_12528_b200 as mp
    rp, ci, v = lap_csr(4, 3, 2)
    n = rp.size - 1
    lines = [(i + 1, ci[p] + 1, float(v[p])) for i in range(n) for p in range(rp[i], rp[i + 1])
             if ci[p] <= i]
    text = ("%%MatrixMarket matrix coordinate REAL Symmetric\n"
            f"{n} {n} {len(lines)}\n" + "".join(f"{i} {j} {x!r}\n" for i, j, x in lines))
    r2, c2, v2 = mp.read_matrix_market(_write(tmp_path, text))
    assert np.array_equal(r2, rp) and np.array_equal(c2, ci) and np.array_equal(v2, v)


@pytest.mark.parametrize("text,exc", [
    ("", "ParseError"),
    ("%%MatrixMarket matrix array real symmetric\n2 2\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n", "NotSymmetricHeader"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1\n", "NotSquare"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n3 1 1\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1\n2 2 1\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 x\n", "ParseError"),
])
def test_errors(tmp_path, text, exc):
    import paper_2302_12528_b200 as mp
    with pytest.raises(getattr(mp, exc)):
        mp.read_matrix_market(_write(tmp_path, text))
