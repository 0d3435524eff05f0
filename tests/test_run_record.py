"""Run reports in the reference's schema (run_record.cpp).  CPU-only.

format_shortest is checked against the reference's own std::to_chars output
(tests/golden/format_shortest.npz, written through oracle/_ref's
mpref_format_shortest); the CSV / JSON layouts follow run_record.cpp:104-160."""
import json

import numpy as np

from conftest import load_golden


def test_format_shortest_matches_reference():
    from paper_2302_12528_b200.run_record import format_shortest
    g = load_golden("format_shortest")
    for v, t in zip(g["vals"], g["text"]):
        assert format_shortest(float(v)) == str(t), (v, t)


def _record(**kw):
    from paper_2302_12528_b200.api import IterationRecord
    from paper_2302_12528_b200.run_record import RunRecord
    h = [IterationRecord(1, [0.5, 1.0], [1e-3, 2e-3], 0, 0, False),
         IterationRecord(0, [0.25, 1.0], [1e-11, 1e-4], 1, 1, True)]
    base = dict(matrix_name="lap3d_32", n=32768, nnz=223232, variant="mplobpcg-schol", k=2,
                m=3, seed=0, iters_lower=1, iters_working=1, converged=True,
                theta=[0.027168464561492175, 0.054254915182245088], resid=[3.5e-15, 1e-04],
                t_factor=0.0, t_total=0.4378, history=h)
    base.update(kw)
    return RunRecord(**base)


def test_csv_rows_per_eigenpair():
    from paper_2302_12528_b200.run_record import BASE_HEADER, run_record_csv
    txt = run_record_csv([_record(), _record(matrix_name="b", converged=False)])
    lines = txt.splitlines()
    assert lines[0] == BASE_HEADER
    assert len(lines) == 1 + 2 + 2
    assert lines[1] == ("lap3d_32,32768,223232,mplobpcg-schol,2,3,0,1,1,1,1,"
                        "0.027168464561492175,3.5e-15,0,0.4378")
    assert lines[2].split(",")[10:13] == ["2", "0.05425491518224509", "1e-04"]
    assert lines[4].split(",")[9] == "0"


def test_history_json_layout():
    from paper_2302_12528_b200.run_record import history_json
    txt = history_json([_record(matrix_name='a"b')])
    d = json.loads(txt)
    assert d[0]["matrix"] == 'a"b' and d[0]["converged"] is True
    it = d[0]["iterations"]
    assert [x["iter"] for x in it] == [1, 2]
    assert [x["stage"] for x in it] == ["lower", "working"]
    assert it[1]["rotation_fallback"] is True and it[1]["w_dropped"] == 1
    assert np.allclose(it[0]["ritz"], [0.5, 1.0])
    assert '"ritz": [0.5,1]' in txt  # format_shortest inside arrays, no spaces
