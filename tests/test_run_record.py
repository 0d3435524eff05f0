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


def _sample(**kw):
    """test_bench.cpp:14-29's sample_record."""
    from paper_2302_12528_b200.run_record import RunRecord
    base = dict(matrix_name="m1", n=4, nnz=16, variant="pinvit", k=2, m=3, seed=9, iters_lower=0,
                iters_working=7, converged=True, theta=[1.5, 2.25], resid=[1e-13, 2e-13])
    base.update(kw)
    return RunRecord(**base)


def test_csv_bound_columns_only_when_present():
    """test_bench.cpp:59-100: the bounded record carries its numbers, the other gets
    11 empty cells, every row has the header's cell count, output deterministic."""
    from paper_2302_12528_b200.analysis import BoundReport
    from paper_2302_12528_b200.run_record import run_record_csv
    recs = [_sample(), _sample(matrix_name="m2", converged=False)]
    a = run_record_csv(recs)
    assert a == run_record_csv(recs) and ",kappa," not in a
    assert a.startswith("matrix,n,nnz,variant,k,m,seed,iters_lower,iters_working,converged,idx,"
                        "theta,resid,t_factor,t_total\nm1,4,16,pinvit,2,3,9,0,7,1,1,1.5,1e-13,0,0\n")
    recs[0].bounds = BoundReport(kappa=100.0, eps_A=1e-14, eps_r=2e-14, eps_T=0.25,
                                 eps_T_vacuous=False, gamma_precond_meas=0.3, norm_te_norm_a=101.0,
                                 beta_mid=4.0, gamma_total_mid=0.31, rate_mid=0.5, floor=1e-12)
    c = run_record_csv(recs)
    assert ",kappa," in c
    assert "1,1.5,1e-13,0,0,100,1e-14,2e-14,0.25,0,0.3,101,4,0.31,0.5,1e-12\n" in c
    assert "1,1.5,1e-13,0,0,,,,,,,,,,,\n" in c
    lines = c.splitlines()
    assert all(l.count(",") == lines[0].count(",") for l in lines)


def test_analysis_bounds_match_reference_cases():
    """The closed-form bounds against test_analysis.cpp's frozen values and guards."""
    import math

    import pytest

    import paper_2302_12528_b200.analysis as an
    u_h, u_l = 2.0 ** -53, 2.0 ** -24
    for n in (1, 2, 100, 1000):
        nu = n * u_h
        assert an.gamma_n(n, u_h) == pytest.approx(nu / (1 - nu), rel=1e-15)
    assert an.gamma_n(1000, u_h) == pytest.approx(1.1102230246251578e-13, rel=1e-12)
    with pytest.raises(an.AssumptionViolated):
        an.gamma_n(1 << 60, 1e-10)
    with pytest.raises(an.AssumptionViolated):
        an.gamma_n(1, -1.0)
    for n in (1, 10, 500):
        assert an.epsilon_A(n, u_h) == pytest.approx(math.sqrt(n) * an.gamma_n(n, u_h), rel=1e-15)
    for n in (5, 50, 200):
        g = n * u_h / (1 - n * u_h)
        ea = math.sqrt(n) * g
        expect = (g + ea + g * ea + (n + 1) * u_h) * (1 + u_h) / (1 - 2 * n * u_h) + ea + u_h
        assert an.epsilon_r(n, u_h, an.epsilon_A(n, u_h)) == pytest.approx(expect, rel=1e-15)
    assert an.epsilon_T(50, 10.0, u_l) == pytest.approx(302000.0 / 16777216.0, rel=1e-15)
    assert an.epsilon_T(10, 100.0, u_l) == pytest.approx(7.390976e-3, rel=1e-6)
    with pytest.raises(an.BoundVacuous):
        an.epsilon_T(100, 1000.0, u_l)
    with pytest.raises(an.AssumptionViolated):
        an.epsilon_T(10, 0.5, u_l)
    e = an.epsilon_T(20, 100.0, u_l)
    assert an.gamma_precond_bound(20, 100.0, u_l) == pytest.approx(e / (1 - e), rel=1e-15)
    assert an.beta(1.5, 1.0, 2.0, 16.0) == pytest.approx(11.313708498, rel=1e-9)
    assert an.beta(1.1, 1.0, 2.0, 16.0) == pytest.approx(40.0, rel=1e-12)
    assert an.beta(1.5, 1.0, 2.0, 2.0) == pytest.approx(4.0, rel=1e-15)
    for args, exc in (((0.5, 1.0, 2.0, 4.0), an.OutOfInterval), ((2.5, 1.0, 2.0, 4.0), an.OutOfInterval),
                      ((1.5, -1.0, 2.0, 4.0), an.AssumptionViolated),
                      ((1.5, 1.0, 2.0, 1.5), an.AssumptionViolated)):
        with pytest.raises(exc):
            an.beta(*args)
    n, g2 = 50, 2 * u_h / (1 - 2 * u_h)
    er = an.epsilon_r(n, u_h, an.epsilon_A(n, u_h))
    assert an.gamma_total(1e-4, 3.0, 20.0, n, u_h, er) == pytest.approx(
        1e-4 + g2 * 3.0 + 20.0 * (u_h + (1 + g2) * er * 3.0), rel=1e-15)
    with pytest.raises(an.AssumptionViolated):
        an.gamma_total(-1e-3, 3.0, 20.0, n, u_h, er)
    assert an.rate_bound(0.0, 1.0, 2.0) == pytest.approx(0.25, rel=1e-15)
    assert an.rate_bound(0.1, 1.0, 10.0) == pytest.approx(0.0361, rel=1e-12)
    assert an.rate_bound(0.999, 1.0, 10.0) < 1.0
    with pytest.raises(an.GammaTooLarge):
        an.rate_bound(1.0, 1.0, 2.0)
    with pytest.raises(an.AssumptionViolated):
        an.rate_bound(0.5, 2.0, 1.0)
    expect = math.sqrt(0.5 * 100.0) * (u_h + (1 + g2) * er * 5.0) / (1 - 1e-3 - g2 * 5.0)
    assert an.accuracy_floor(1e-3, 5.0, n, u_h, er, 0.5, 100.0) == pytest.approx(expect, rel=1e-15)
    assert an.accuracy_floor(1e-3, 5.0, n, u_h, er, 0.5, 100.0) < 1e-11
    with pytest.raises(an.DenominatorNonpositive):
        an.accuracy_floor(1.0, 5.0, n, u_h, er, 0.5, 100.0)
    D = np.diag([3.0, 0.5, 7.5, 1.0])
    assert an.operator_norm_2(D) == pytest.approx(7.5, rel=1e-12)
