"""North-star configurations on one GPU (GPU box helper):

    python scripts/cfg_run.py cfg2 --capped 40 --full > gpurun_out/r02_cfg2.json
    python scripts/cfg_run.py cfg4 --capped 12            > gpurun_out/r02_cfg4_1gpu.json

cfg2: 2-D 5-pt Laplacian 1024^2 (n = 1,048,576), k = 32, m = 48, Jacobi f_T:
      MPLOBPCG-schol (to tol 1e-10 with --full) and PINVIT (capped).
cfg4: 3-D 7-pt Laplacian 256^3 (n = 16,777,216), k = 64, m = 80, Jacobi f_T.
A capped solve gives iterations/s and the per-kernel shares (profiling pass);
--full solves to the tolerance and checks theta against the analytic Dirichlet
spectrum (sums of 4 sin^2(i pi / (2 (N + 1))), the 3-D analogue of
generators.cpp:32-46).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2302_12528_b200 as mp  # noqa: E402

CFGS = {
    "cfg2": dict(dims=(1024, 1024), k=32, block=48),
    "cfg4": dict(dims=(256, 256, 256), k=64, block=80),
    "cfg4_half": dict(dims=(256, 256, 128), k=64, block=80),
    "lap3d128": dict(dims=(128, 128, 128), k=32, block=48),
    # cfg5: Kohn-Sham-like -Laplacian + V (seeded wells), n = 4,194,304, k = 128
    "cfg5": dict(dims=(256, 128, 128), k=128, block=192, ks=True),
    "ks64": dict(dims=(64, 64, 64), k=32, block=48, ks=True),
}


def analytic(dims, k):
    lam1 = [4 * np.sin(np.arange(1, min(N, k + 1) + 1) * np.pi / (2 * (N + 1))) ** 2 for N in dims]
    tot = lam1[0]
    for l in lam1[1:]:
        tot = np.add.outer(tot, l).ravel()
    return np.sort(tot)[:k]


def op(dims, ks=False):
    if ks:
        return mp.ks_hamiltonian(*dims, seed=0)
    return mp.laplace2d(*dims) if len(dims) == 2 else mp.laplace3d(*dims)


def capped(name, variant, iters):
    """Per-iteration time from two capped solves (iters and 2 iters per stage):
    the difference cancels the setup (host RNG draws of the start block and
    sketch, norm estimate, initial QR, allocation)."""
    c = CFGS[name]
    A = op(c["dims"], c.get("ks", False))
    import torch

    def timed(maxit):
        cfg = mp.SolverConfig(k=c["k"], block=c["block"], tol=1e-10, maxit=maxit, variant=variant)
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = mp.solve(A, cfg, want_X=False, history=False)
        torch.cuda.synchronize()
        return time.perf_counter() - t, r.iterations_lower + r.iterations_working, r

    timed(iters)  # warm-up: allocations, graphs
    t1, i1, _ = timed(iters)
    t2, i2, r = timed(2 * iters)
    dt, di = t2 - t1, i2 - i1
    cfg = mp.SolverConfig(k=c["k"], block=c["block"], tol=1e-10, maxit=iters, variant=variant)
    with mp.profile():
        mp.solve(A, cfg, want_X=False, history=False)
        torch.cuda.synchronize()
        rep = mp.profile.report()
    tot = sum(v["ms"] for v in rep.values()) or 1.0
    kern = {}
    for nm, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
        if v["count"] == 0:
            continue
        kern[nm] = {"launches": v["count"], "share": round(v["ms"] / tot, 4),
                    "ms_per_launch": round(v["ms"] / v["count"], 4),
                    "GBps": round(v["bytes"] / (v["ms"] * 1e6), 1) if v["bytes"] > 0 and v["ms"] > 0 else None,
                    "TFps": round(v["flops"] / (v["ms"] * 1e9), 2) if v["flops"] > 0 and v["ms"] > 0 else None}
    # per-stage iteration times from the host arrival of the per-iteration records
    cfg2 = mp.SolverConfig(k=c["k"], block=c["block"], tol=1e-10, maxit=2 * iters, variant=variant)
    rh = mp.solve(A, cfg2, want_X=False, history=True)
    per_stage = {}
    h = rh.history
    for st in sorted({x.stage for x in h}):
        ts = [x.host_time for x in h if x.stage == st]
        if len(ts) > 2:
            d = np.diff(ts)[1:]  # skip the stage's first (setup) interval
            per_stage["fp32" if st == 1 else "fp64"] = {"ms_per_iteration_median": 1e3 * float(np.median(d)),
                                                        "iterations": len(d)}
    return {"variant": variant, "iterations": [r.iterations_lower, r.iterations_working],
            "per_stage_from_records": per_stage,
            "method": f"(t[{2 * iters}/stage] - t[{iters}/stage]) / extra iterations",
            "ms_per_iteration": 1e3 * dt / max(di, 1), "iters_per_s": di / dt,
            "kernels_profiling_pass": kern}


def full(name, variant, maxit):
    c = CFGS[name]
    A = op(c["dims"], c.get("ks", False))
    cfg = mp.SolverConfig(k=c["k"], block=c["block"], tol=1e-10, maxit=maxit, variant=variant)
    import torch
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = mp.solve(A, cfg, want_X=False, history=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if c.get("ks"):
        err = np.full(c["k"], np.nan)  # no closed form for -Laplacian + V
    else:
        lam = analytic(c["dims"], c["k"])
        err = np.abs(r.theta - lam) / lam
    thr = 1e-10 * (r.a_norm_estimate + np.abs(r.theta))
    h = r.history
    trace = [{"it": i, "stage": int(h[i].stage), "n_c": int(h[i].n_converged),
              "max_resid": float(np.max(h[i].residual_norms[:c["k"]]))}
             for i in range(0, len(h), max(1, len(h) // 40))]
    its = r.iterations_lower + r.iterations_working
    return {"variant": variant, "converged": r.converged,
            "iterations": [r.iterations_lower, r.iterations_working], "time_to_solution_s": dt,
            "iters_per_s": its / dt, "theta_max_rel_err_vs_analytic": float(err.max()),
            "residual_contract": bool(np.all(r.residual_norms <= thr * (1 + 1e-12))),
            "a_norm_est": r.a_norm_estimate, "theta": r.theta.tolist(), "trace": trace,
            "timings": vars(r.timings)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", choices=sorted(CFGS))
    ap.add_argument("--capped", type=int, default=0)
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--maxit", type=int, default=30000)
    ap.add_argument("--variants", default="mplobpcg-schol,dlobpcg-dchol")
    ap.add_argument("--pinvit", type=int, default=0, help="capped PINVIT iterations")
    a = ap.parse_args()
    c = CFGS[a.cfg]
    out = {"config": a.cfg, "dims": c["dims"], "k": c["k"], "block": c["block"], "tol": 1e-10,
           "precond": "Jacobi (fp32 f_T)", "gpu": None}
    try:
        import torch
        out["gpu"] = torch.cuda.get_device_name(0)
    except Exception:
        pass
    variants = [v for v in a.variants.split(",") if v]
    if a.capped:
        out["capped"] = [capped(a.cfg, v, a.capped) for v in variants]
        print(json.dumps(out["capped"][-1]["ms_per_iteration"]), file=sys.stderr, flush=True)
    if a.pinvit:
        out["pinvit_capped"] = capped(a.cfg, "pinvit", a.pinvit)
    if a.full:
        out["full"] = []
        for v in variants:
            out["full"].append(full(a.cfg, v, a.maxit))
            print(json.dumps({k: out["full"][-1][k] for k in ("variant", "iterations", "time_to_solution_s")}),
                  file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
