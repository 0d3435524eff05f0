"""Run reports in the reference's schema: RunRecord
(run_record.hpp:16-32) flattened to CSV (run_record.cpp:104-116, one row per
eigenpair, run-level fields repeated) and the per-iteration history as JSON
(:124-160), numbers in shortest round-trip form exactly as std::to_chars writes
them (format_shortest, :97-102), so GPU and CPU reports diff cleanly.

Host-side reporting.  A record may carry an analysis.BoundReport (the reference
CLI's --bounds, analysis.cpp / bench_main.cpp:116-171); the CSV then grows the
bound columns (run_record.cpp:14-16, 50-66), with empty cells for records
without bounds.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

BASE_HEADER = ("matrix,n,nnz,variant,k,m,seed,iters_lower,iters_working,converged,idx,"
               "theta,resid,t_factor,t_total")
BOUNDS_HEADER = (",kappa,eps_A,eps_r,eps_T,eps_T_vacuous,gamma_precond,norm_te_norm_a,"
                 "beta_mid,gamma_total_mid,rate_mid,floor")


def format_shortest(v: float) -> str:
    """std::to_chars(double) with no format: the shortest round-trip digits, written
    fixed or scientific, whichever is shorter (fixed on a tie); exponent >= 2 digits;
    an integral value in fixed form is its exact decimal expansion."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    # shortest round-trip digits and decimal exponent from repr
    mant, _, exp = repr(abs(v)).partition("e")
    e = int(exp) if exp else 0
    ip, _, fp = mant.partition(".")
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0")
    lead_zeros = len(ip + fp) - len((ip + fp).lstrip("0"))
    e10 = e + len(ip) - 1 - lead_zeros  # exponent of the first significant digit
    digits = digits.rstrip("0") or "0"
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "")
    sci += "e" + ("-" if e10 < 0 else "+") + f"{abs(e10):02d}"
    if e10 >= 0:
        if len(digits) <= e10 + 1:
            # an integral value: %f writes its exact decimal expansion
            fixed = str(int(abs(v)))
        else:
            fixed = digits[:e10 + 1] + "." + digits[e10 + 1:]
    else:
        fixed = "0." + "0" * (-e10 - 1) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


@dataclass
class RunRecord:
    """run_record.hpp:16-32."""
    matrix_name: str
    n: int
    nnz: int
    variant: str
    k: int
    m: int
    seed: int
    iters_lower: int
    iters_working: int
    converged: bool
    theta: List[float]
    resid: List[float]
    t_factor: float = 0.0
    t_total: float = 0.0
    history: list = field(default_factory=list)
    bounds: Optional[object] = None

    @classmethod
    def from_result(cls, name: str, n: int, nnz: int, cfg, r, t_factor: float = 0.0,
                    t_total: float = 0.0) -> "RunRecord":
        """From an api.EigResult and its SolverConfig."""
        return cls(name, n, nnz, cfg.variant, cfg.k, cfg.block_size(), cfg.seed,
                   r.iterations_lower, r.iterations_working, r.converged,
                   [float(x) for x in r.theta], [float(x) for x in r.residual_norms],
                   t_factor, t_total if t_total else getattr(r.timings, "total", 0.0),
                   list(r.history))


def _bound_cells(b) -> str:
    """The 11 bound cells of one row (run_record.cpp:50-66); empty without bounds."""
    if b is None:
        return "," * 11
    cells = [format_shortest(v) for v in (b.kappa, b.eps_A, b.eps_r, b.eps_T)]
    cells.append("1" if b.eps_T_vacuous else "0")
    cells += [format_shortest(v) for v in (b.gamma_precond_meas, b.norm_te_norm_a, b.beta_mid,
                                           b.gamma_total_mid, b.rate_mid, b.floor)]
    return "," + ",".join(cells)


def run_record_csv(records: List[RunRecord]) -> str:
    """run_record_csv (run_record.cpp:104-116); bound columns only when a record has them."""
    with_bounds = any(r.bounds is not None for r in records)
    out = [BASE_HEADER + (BOUNDS_HEADER if with_bounds else "") + "\n"]
    for r in records:
        for j in range(len(r.theta)):
            out.append(",".join([
                r.matrix_name, str(r.n), str(r.nnz), r.variant, str(r.k), str(r.m), str(r.seed),
                str(r.iters_lower), str(r.iters_working), "1" if r.converged else "0", str(j + 1),
                format_shortest(r.theta[j]), format_shortest(r.resid[j]),
                format_shortest(r.t_factor), format_shortest(r.t_total)]) +
                (_bound_cells(r.bounds) if with_bounds else "") + "\n")
    return "".join(out)


def _json_str(s: str) -> str:
    o = ['"']
    for ch in s:
        if ch in '"\\':
            o.append("\\" + ch)
        elif ord(ch) < 0x20:
            o.append(" ")
        else:
            o.append(ch)
    o.append('"')
    return "".join(o)


def _json_arr(v) -> str:
    return "[" + ",".join(format_shortest(x) for x in v) + "]"


def history_json(records: List[RunRecord]) -> str:
    """history_json (run_record.cpp:124-160); history entries are api.IterationRecord."""
    out = ["[\n"]
    for ri, rec in enumerate(records):
        out.append("  {\"matrix\": " + _json_str(rec.matrix_name) + ", \"variant\": " +
                   _json_str(rec.variant) + f", \"seed\": {rec.seed}, \"converged\": " +
                   ("true" if rec.converged else "false") + ", \"iterations\": [\n")
        for i, it in enumerate(rec.history):
            stage = "\"lower\"" if getattr(it, "stage", "working") in ("lower", 1) else "\"working\""
            out.append(f"    {{\"iter\": {i + 1}, \"stage\": {stage}, \"n_converged\": "
                       f"{it.n_converged}, \"w_dropped\": {it.w_columns_dropped}, "
                       "\"rotation_fallback\": " +
                       ("true" if it.basis_rotation_fallback else "false") +
                       ", \"ritz\": " + _json_arr(it.ritz_values) + ", \"resid\": " +
                       _json_arr(it.residual_norms) + "}" +
                       ("," if i + 1 < len(rec.history) else "") + "\n")
        out.append("  ]}" + ("," if ri + 1 < len(records) else "") + "\n")
    out.append("]\n")
    return "".join(out)


def write_csv(path: str, records: List[RunRecord]) -> None:
    with open(path, "w") as f:
        f.write(run_record_csv(records))


def write_history_json(path: str, records: List[RunRecord]) -> None:
    with open(path, "w") as f:
        f.write(history_json(records))
