"""cfg3 (BASELINE.json configs[2]): dense SPD n = 16384 with a prescribed
log-spaced spectrum in [1, kappa], k = 64 (m = 96), tol 1e-10, solved with the
reference's stock dense path -- solve(DenseMatrix, cfg) with its Cholesky
preconditioner (drivers.hpp:158-181, precond.hpp:33-50) -- on one B200.

A = H1 H2 H3 diag(lam) H3 H2 H1 (the spd_dense recipe of tests/problems.py:
same seeded lam and reflectors, the reflectors applied two-sided on the device
at O(n^2) each instead of forming Q).  The spectrum is known, so the computed
theta is checked against lam[:k] at full size.

    python scripts/cfg3_dense.py [n] [k] [kappa]
Prints one JSON line per variant: factor time, solve time (wall clock around
the synchronous call = device time: the library syncs once per iteration),
iterations, it/s, max |theta - lam| / lam, per-kernel-class shares of a
profiled solve.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_12528_b200 as mp  # noqa: E402


def build(n, kappa, seed):
    rng = np.random.default_rng(seed)
    lam = np.sort(np.exp(np.log(kappa) * rng.random(n)))
    lam[0], lam[-1] = 1.0, kappa
    vs = [rng.standard_normal(n) for _ in range(3)]
    A = torch.diag(torch.tensor(lam, dtype=torch.float64, device="cuda"))
    for v in reversed(vs):  # Q = H1 H2 H3: innermost reflector first
        v = torch.tensor(v, dtype=torch.float64, device="cuda")
        vv = float(v @ v)
        w = A @ v
        vw = float(v @ w)
        A -= (2.0 / vv) * (torch.outer(v, w) + torch.outer(w, v))
        A += (4.0 * vw / (vv * vv)) * torch.outer(v, v)
    A = 0.5 * (A + A.T)
    return np.asfortranarray(A.cpu().numpy()), lam


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    kappa = float(sys.argv[3]) if len(sys.argv) > 3 else 1e3
    t0 = time.perf_counter()
    Ah, lam = build(n, kappa, 5)
    t_gen = time.perf_counter() - t0
    A = mp.dense_matrix(Ah)
    del Ah
    for variant in ("mplobpcg-schol", "dlobpcg-dchol"):
        cfg = mp.SolverConfig(variant=variant, k=k, tol=1e-10, maxit=1000, seed=0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        T = mp.dense_cholesky(A, mp.build_precision_for(variant))
        torch.cuda.synchronize()
        t_fac = time.perf_counter() - t0
        mp.solve(A, cfg, T=T, want_X=False, history=False)  # warm-up
        times = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = mp.solve(A, cfg, T=T, want_X=False, history=False)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        with mp.profile():
            mp.solve(A, cfg, T=T, want_X=False, history=False)
        rep = mp.profile.report()
        tot = sum(v["ms"] for v in rep.values()) or 1.0
        kern = {}
        for name, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
            e = {"launches": v["count"], "share": round(v["ms"] / tot, 4),
                 "ms_per_launch": round(v["ms"] / max(v["count"], 1), 4)}
            if v["ms"] > 0 and v["flops"] > 0:
                e["TFps"] = round(v["flops"] / v["ms"] / 1e9, 2)
            if v["ms"] > 0 and v["bytes"] > 0:
                e["GBps"] = round(v["bytes"] / v["ms"] / 1e6, 1)
            kern[name] = e
        it = r.iterations_lower + r.iterations_working
        t = min(times)
        print(json.dumps({
            "workload": f"cfg3: dense SPD n={n}, log-spaced spectrum [1, {kappa:g}], k={k}, "
                        f"m={cfg.block_size()}, tol 1e-10, dense Cholesky f_T",
            "variant": variant, "converged": r.converged,
            "iterations": {"lower": r.iterations_lower, "working": r.iterations_working},
            "factor_s": round(t_fac, 4), "solve_s": round(t, 4),
            "solve_s_runs": [round(x, 4) for x in times], "iters_per_s": round(it / t, 1),
            "theta_max_rel_err_vs_spectrum": float(np.max(np.abs(r.theta - lam[:k]) / lam[:k])),
            "precond_shift": T.shift, "generate_s": round(t_gen, 2), "kernels": kern}),
            flush=True)


if __name__ == "__main__":
    main()
