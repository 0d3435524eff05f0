#!/usr/bin/env python
"""bench.py -- LOBPCG time-to-solution of the B200 (sm_100a) path vs the reference.

Workload (N=1): BASELINE.json configs[0] / BASELINE.md §2 ("cfg1"): 3-D 7-point
Laplacian 32^3 (n = 32,768), k = 10, m = 16, tol 1e-10, Jacobi f_T, seed 0,
mixed precision (MPLOBPCG-schol: fp32 stage to 5e-6, then fp64 with mixed_qr).
This is the only configuration whose time-to-solution the reference can be
measured on (configs[1] at tol 1e-10 needs >1e4 unpreconditioned iterations;
see DESIGN.md §Measurement).  A "step" is one complete solve.

    python bench.py                        # N=1, 5 timed solves after 3 warm-ups
    python bench.py --impl reference       # the reference CPU solver (oracle/_ref):
                                           # K complete solves, side by side on the host cores
    torchrun --nproc-per-node N bench.py --gpus N   # ONE row-sharded solve over the N GPUs
    torchrun --nproc-per-node N bench.py --gpus N --replicas   # N independent replicas

Prints ONE JSON line (rank 0).  `value` = mean device time of one solve with
all inputs resident in HBM (seconds, lower is better); `e2e` = the same solve
through the C ABI with the start block / sketch copied from pinned host memory
and the eigenvectors copied back inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "cfg1": dict(dims=(32, 32, 32), k=10, block=16, tol=1e-10, maxit=2000, seed=0,
                 desc="3-D 7-pt Laplacian 32^3 (n=32768), k=10, m=16, tol 1e-10, Jacobi f_T"),
    # larger row-sharded workloads (bench.py --shard under torchrun)
    "lap3d128": dict(dims=(128, 128, 128), k=32, block=48, tol=1e-10, maxit=20000, seed=0,
                     desc="3-D 7-pt Laplacian 128^3 (n=2.1M), k=32, m=48, tol 1e-10, Jacobi f_T"),
    "cfg4": dict(dims=(256, 256, 256), k=64, block=80, tol=1e-10, maxit=20000, seed=0,
                 desc="3-D 7-pt Laplacian 256^3 (n=16.8M), k=64, m=80, tol 1e-10, Jacobi f_T"),
}
METRIC = "LOBPCG time-to-solution (k eigpairs, tol 1e-10)"
REF_SAMPLE_ITERS = 10  # per stage, per reference sample


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def golden_iters(workload, variant):
    p = os.path.join(ROOT, "tests", "golden", f"{workload}-{variant}.npz")
    if not os.path.exists(p):
        return None
    g = np.load(p)
    return {"lower": int(g["iters_lower"]), "working": int(g["iters_working"]),
            "theta": g["theta"], "t_total": float(g["t_total"])}


# --------------------------------------------------------------- reference arm
def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    if hasattr(os, "sched_getaffinity"):
        avail = sorted(os.sched_getaffinity(0))
    else:
        avail = list(range(os.cpu_count() or 1))
    return {"cpu_model": model, "nproc": os.cpu_count(), "usable_cores": len(avail)}, avail


def _ref_worker(args):
    """One unmodified reference solve (oracle/_ref: the reference library through
    its own lobpcg_stage / BlockOperator API), pinned to one host core."""
    workload, variant, core, maxit = args
    if core is not None and hasattr(os, "sched_setaffinity"):
        os.sched_setaffinity(0, {core})
    from oracle import Oracle, Problem, available
    w = WORKLOADS[workload]
    which = "ref" if available("ref") else "port"
    t0 = time.perf_counter()
    r = Oracle(which).solve(Problem.lap3d(*w["dims"]), variant, k=w["k"], block=w["block"],
                            tol=w["tol"], maxit=maxit or w["maxit"], seed=w["seed"], hist_cap=0)
    wall = time.perf_counter() - t0
    return {"t_solve": r.t_total, "wall": wall, "iters": [r.iters_lower, r.iters_working],
            "converged": r.converged, "theta": r.theta.tolist(),
            "kind": "reference" if which == "ref" else "port"}


def reference_full_solves(workload, variant, count, maxit=None):
    """`count` complete reference solves run side by side, one per host core (in
    waves when count exceeds the usable cores; one core is left free).  Each
    solve is single-threaded, as the reference is; running them
    concurrently is how the reference arm uses the host's threads.  Returns the
    per-solve results, the batch's wall time, host info and the concurrency."""
    import multiprocessing as mpc
    info, cores = host_info()
    slots = cores[1:] if len(cores) > 1 else cores
    jobs = [(workload, variant, slots[i % len(slots)], maxit) for i in range(count)]
    conc = min(count, len(slots))
    t0 = time.perf_counter()
    with mpc.get_context("spawn").Pool(conc) as pool:
        res = pool.map(_ref_worker, jobs, chunksize=1)
    return res, time.perf_counter() - t0, info, conc


def reference_summary(workload, variant, res, wall, info, conc):
    gi = golden_iters(workload, variant)
    t = np.array([r["t_solve"] for r in res])
    its = res[0]["iters"]
    err = None
    if gi is not None:
        err = max(float(np.max(np.abs(np.array(r["theta"]) - gi["theta"]) / np.abs(gi["theta"])))
                  for r in res)
    return {
        "value": float(np.median(t)), "best": float(t.min()), "worst": float(t.max()),
        "solves": len(res), "concurrent": conc, "batch_wall_s": wall,
        "iterations": {"lower": its[0], "working": its[1]},
        "all_iterations_identical": all(r["iters"] == its for r in res),
        "golden_iterations": {"lower": gi["lower"], "working": gi["working"]} if gi else None,
        "theta_max_rel_err_vs_golden": err, "converged": all(r["converged"] for r in res),
        "host": info, "kind": res[0]["kind"],
    }


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    # warm-up: W short (capped) solves page in the library and the host caches
    for _ in range(args.warmup):
        _ref_worker((args.workload, args.variant, None, 5))
    res, wall, info, conc = reference_full_solves(args.workload, args.variant, args.steps)
    sm = reference_summary(args.workload, args.variant, res, wall, info, conc)
    value = sm["value"]
    sample = (f"{sm['solves']} complete reference solves to tol {w['tol']} "
              f"({sm['iterations']['lower']}+{sm['iterations']['working']} iterations each), "
              f"{conc} side by side, one per host core; value = median time-to-solution "
              f"(best {sm['best']:.1f} s, worst {sm['worst']:.1f} s)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # the K solves ran side by side: the timed region is the batch's wall time
        "ms_per_step": wall * 1e3 / args.steps,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": dtype_of(args.variant),
        "data": "synthetic (deterministic Laplacian, seeded PCG64 start block)",
        "config": {"workload": f"{args.workload}: {w['desc']}", "variant": args.variant},
        "cpu_baseline": {"value": value, "unit": "s", "cores": 1, "kind": sm["kind"], "sample": sample},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_run": sm,
    }
    print(json.dumps(line), flush=True)


def reference_sample_estimate(workload, variant):
    """Cross-check only: a 10+10-iteration sample of the reference scaled to its
    golden iteration counts (never reported as a measured value)."""
    from oracle import Oracle, Problem, available
    w = WORKLOADS[workload]
    which = "ref" if available("ref") else "port"
    r = Oracle(which).solve(Problem.lap3d(*w["dims"]), variant, k=w["k"], block=w["block"],
                            tol=w["tol"], maxit=REF_SAMPLE_ITERS, seed=w["seed"], hist_cap=0)
    gi = golden_iters(workload, variant)
    t1 = r.extra.get("t_stage1", 0.0)
    t_hi = r.t_total - r.t_setup - t1
    full_lo, full_hi = (gi["lower"], gi["working"]) if gi else (r.iters_lower, r.iters_working)
    return (r.t_setup + (t1 / max(r.iters_lower, 1)) * full_lo
            + (t_hi / max(r.iters_working, 1)) * full_hi)


def dtype_of(variant):
    return {"mplobpcg-schol": "f64+f32", "dlobpcg-schol": "f64 (f32 f_T)",
            "dlobpcg-dchol": "f64", "pinvit": "f64 (f32 f_T)"}[variant]


# --------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import paper_2302_12528_b200 as mp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # a fixed NCCL algorithm / protocol keeps the allreduce summation order
        # (and so the sharded trajectory) reproducible run to run
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    w = WORKLOADS[args.workload]
    # N > 1: one row-sharded solve over the N GPUs (SURVEY §8e, strong scaling)
    # unless --replicas; at N = 1 --shard runs the sharded path over a 1-rank comm
    shard = args.shard or (world > 1 and not args.replicas)
    ctx = mp.Context(local)
    cfg = mp.SolverConfig(k=w["k"], block=w["block"], tol=w["tol"], maxit=w["maxit"], seed=w["seed"],
                          variant=args.variant)
    m, k, sr = cfg.block_size(), cfg.k, cfg.sketch_rows
    if shard:
        # row-sharded solve: rank r owns z-slab r; Gram / norm
        # allreduce, R allgather and halo planes over NCCL (NVLink / NVSwitch)
        ctx.attach_nccl(rank, world,
                        mp.broadcast_unique_id(rank) if world > 1 else mp.nccl_unique_id())
        nx, ny, nz = w["dims"]
        z0, nzl = mp.slab_partition(nz, world)[rank]
        A = mp.laplace3d_slab(nx, ny, nz, z0, nzl, ctx=ctx)
        n_glob, row0 = nx * ny * nz, nx * ny * z0
    else:
        A = mp.laplace3d(*w["dims"], ctx=ctx)
        n_glob, row0 = A.n, 0
    T = mp.jacobi(A, mp.build_precision_for(args.variant))
    n = A.n
    dev = f"cuda:{local}"

    # inputs: gaussian_matrix(n, m, seed) and the sketch Omega (this rank's
    # rows when sharded), drawn once on the host
    if shard:
        X0h = mp.gaussian_matrix_rows(n_glob, m, cfg.seed, row0, n)
        Omh = mp.gaussian_matrix_rows(n_glob, sr, cfg.seed ^ 0x9E3779B97F4A7C15, row0, n)
        om_fro = 0.0  # ||Omega||_F reduced over the ranks on the device
    else:
        X0h = mp.gaussian_matrix(n, m, cfg.seed)
        Omh = mp.gaussian_matrix(n, sr, cfg.seed ^ 0x9E3779B97F4A7C15)
        om_fro = float(np.sqrt(np.sum(np.abs(Omh.ravel(order="F")) ** 2)))
    X0pin = torch.from_numpy(np.ascontiguousarray(X0h.T)).pin_memory()
    Ompin = torch.from_numpy(np.ascontiguousarray(Omh.T)).pin_memory()
    X0d, Omd = X0pin.to(dev), Ompin.to(dev)
    Xout = torch.empty((k, n), dtype=torch.float64, device=dev)
    Xhost = torch.empty((k, n), dtype=torch.float64).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 2x L2
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def solve_resident():
        return mp.solve_prepared(A, cfg, X0d, Omd, om_fro, T=T, X_out=Xout)

    def solve_e2e():
        xd = X0pin.to(dev, non_blocking=True)
        od = Ompin.to(dev, non_blocking=True)
        r = mp.solve_prepared(A, cfg, xd, od, om_fro, T=T, X_out=Xout)
        Xhost.copy_(Xout, non_blocking=True)
        stream.synchronize()
        return r

    for _ in range(args.warmup):
        r = solve_resident()
    # ---- timed region (inputs resident)
    times, iters = [], []
    launches0 = ctx.launches()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = solve_resident()
            e1.record(stream)
            barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
            iters.append((r.iterations_lower, r.iterations_working))
    launches = ctx.launches() - launches0
    t_step = float(np.mean(times))
    # ---- e2e through the C ABI with host buffers
    e2e_times = []
    for _ in range(max(2, args.steps // 2)):
        flush.fill_(1.0)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        r_e2e = solve_e2e()
        e1.record(stream)
        barrier()
        e2e_times.append(max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0))
    t_e2e = float(np.mean(e2e_times))
    if dist:
        t = torch.tensor([t_step, t_e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step, t_e2e = t.tolist()
    # ---- roofline: one instrumented solve (CUDA events around every launch)
    with mp.profile():
        solve_resident()
        torch.cuda.synchronize()
        prof = mp.profile.report()
    # ---- the north-star target's per-iteration time at this N (cfg4: 256^3,
    # k = 64, m = 80, row-sharded over the N GPUs; evidence key, all ranks)
    at_scale = {}
    if (world > 1 or args.cfg4) and not args.no_at_scale and args.workload == "cfg1" and not args.replicas:
        for which in ("cfg4", "cfg5"):
            try:
                at_scale[which] = cfg4_per_iteration(mp, ctx, rank, world, dist, shard, which=which)
            except Exception as exc:  # evidence only: never fail the bench line
                at_scale[which] = {"error": f"{type(exc).__name__}: {exc}"}
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = load_peaks()
    tot_ms = sum(v["ms"] for v in prof.values()) or 1.0
    kernels = {}
    for name, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        c = max(v["count"], 1)
        kernels[name] = {"launches": v["count"], "share": round(v["ms"] / tot_ms, 4),
                         "us_per_launch": round(1e3 * v["ms"] / c, 3),
                         "GBps": round(v["bytes"] / (v["ms"] * 1e6), 1) if v["ms"] > 0 and v["bytes"] > 0 else None}
    # the roofline kernel: the largest-share bandwidth-bound family that has an ncu
    # DRAM capture (profiles/ncu_traffic.json: the fp64 Gram family at cfg1 -- the
    # fp32 and fp64 Grams are separate families and share the top place), else the
    # largest-share bandwidth-bound family
    captured = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            captured = json.load(f).get(args.workload, {})
    bw = [nme for nme in kernels if prof[nme]["bytes"] > 0]
    top = next((nme for nme in bw if nme in captured), bw[0] if bw else None)
    roof = None
    if top:
        v = prof[top]
        c = max(v["count"], 1)
        achieved = (v["bytes"] / c) / ((v["ms"] / c) * 1e6)
        traffic = captured.get(top)
        roof = {"kernel": top, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "algorithmic_bytes_per_launch": v["bytes"] / c,
                "launches": v["count"], "share_of_solve": kernels[top]["share"]}
    gi = golden_iters(args.workload, args.variant)
    cpu = None
    if world == 1 and not args.no_cpu_baseline and args.workload == "cfg1":
        # the reference on the host cores, after the GPU timing: 3 complete
        # solves side by side (best of 3 reported), CPU model and core count
        res, wall, info, conc = reference_full_solves(args.workload, args.variant, 3)
        sm = reference_summary(args.workload, args.variant, res, wall, info, conc)
        cpu = {"value": sm["best"], "unit": "s", "cores": 1, "kind": sm["kind"],
               "sample": (f"best of {sm['solves']} complete reference solves ({conc} side by side, one "
                          f"per host core, {sm['iterations']['lower']}+{sm['iterations']['working']} "
                          f"iterations each); median {sm['value']:.1f} s"),
               "reference_run": sm,
               "estimate_from_10_iteration_sample": reference_sample_estimate(args.workload, args.variant)}
    theta_err = None
    if gi is not None:
        theta_err = float(np.max(np.abs(r.theta - gi["theta"]) / np.abs(gi["theta"])))
    line = {
        "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False,
        "scaling": "strong" if shard else "weak", "vs_baseline": None,
        "dtype": dtype_of(args.variant),
        "data": "synthetic (deterministic Laplacian, seeded PCG64 start block)",
        "config": {"workload": f"{args.workload}: {w['desc']}", "variant": args.variant,
                   "l2": "flushed (256 MB write) before every solve",
                   "parallelism": (f"row-sharded over {world} GPUs (NCCL)" if shard else
                                   "replicas" if world > 1 else "single GPU"),
                   "iterations": {"lower": iters[-1][0], "working": iters[-1][1]},
                   "reference_iterations": {"lower": gi["lower"], "working": gi["working"]} if gi else None,
                   "theta_max_rel_err_vs_reference": theta_err,
                   "iters_per_s": (iters[-1][0] + iters[-1][1]) / t_step},
        "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": 8 * n * (m + sr),
                "d2h_bytes_per_step": 8 * n * k + 16 * k},
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    if world == 1 and not shard and args.workload == "cfg1" and not args.no_at_scale:
        try:
            line["kernels_at_scale"] = at_scale_kernels(mp, peak)
        except Exception as exc:  # evidence only: never fail the bench line
            line["kernels_at_scale"] = {"error": f"{type(exc).__name__}: {exc}"}
    for which, v in at_scale.items():
        line[f"{which}_per_iteration"] = v
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


DMMA_PEAK_TFS = 37.1  # fp64 mma.sync m8n8k4, measured in-repo (profiles/r01_microbench_b200.txt)
BF16_PEAK_TFS = 2150.0  # tcgen05 kind::f16 M=128 N=160 issue rate, scripts/micro/umma_rate.cu
TC_FAMILIES = ("gram_f32", "gemm_f32")


AT_SCALE = {
    "cfg4": dict(dims=(256, 256, 256), k=64, m=80, ks=False,
                 desc="cfg4: 3-D 7-pt Laplacian 256^3 (n=16.8M), k=64, m=80"),
    "cfg5": dict(dims=(256, 128, 128), k=128, m=192, ks=True,
                 desc="cfg5: Kohn-Sham-like -Laplacian+V 256x128x128 (n=4.2M), k=128, m=192"),
}


def cfg4_per_iteration(mp, ctx, rank, world, dist, shard, iters=4, which="cfg4"):
    """BASELINE.json configs[3] (cfg4: 3-D 7-pt Laplacian 256^3, k = 64, m = 80)
    or configs[4] (cfg5: the Kohn-Sham-like operator, n = 4.2M, k = 128) at
    this N: mixed precision, row-sharded over the N GPUs (z-slabs, overlapped
    halo exchange, Gram / norm allreduce over NCCL); a capped solve (`iters`
    per stage).  Per-iteration time = median interval between the
    per-iteration records reaching the host, per stage, max over ranks.  A
    full solve to 1e-10 takes thousands of iterations."""
    import torch
    w = AT_SCALE[which]
    nx, ny, nz = w["dims"]
    k, m = w["k"], w["m"]
    cfg = mp.SolverConfig(k=k, block=m, tol=1e-10, maxit=iters, variant="mplobpcg-schol")
    if shard:
        z0, nzl = mp.slab_partition(nz, world)[rank]
        A = (mp.ks_hamiltonian_slab(nx, ny, nz, z0, nzl, seed=0, ctx=ctx) if w["ks"] else
             mp.laplace3d_slab(nx, ny, nz, z0, nzl, ctx=ctx))
        row0 = nx * ny * z0
    else:
        A = mp.ks_hamiltonian(nx, ny, nz, seed=0, ctx=ctx) if w["ks"] else mp.laplace3d(nx, ny, nz, ctx=ctx)
        row0 = 0
    n_glob, n = nx * ny * nz, A.n
    dev = f"cuda:{ctx.device}"
    X0 = torch.from_numpy(np.ascontiguousarray(
        mp.gaussian_matrix_rows(n_glob, m, cfg.seed, row0, n).T)).to(dev)
    Om = torch.from_numpy(np.ascontiguousarray(
        mp.gaussian_matrix_rows(n_glob, cfg.sketch_rows, cfg.seed ^ 0x9E3779B97F4A7C15, row0, n).T)).to(dev)
    T = mp.jacobi(A, mp.LOWER)
    mp.solve_prepared(A, cfg, X0, Om, 0.0, T=T)  # warm-up: allocations
    torch.cuda.synchronize()
    r = mp.solve_prepared(A, cfg, X0, Om, 0.0, T=T, history=True)
    torch.cuda.synchronize()
    med = []
    for st in (1, 0):  # fp32 stage, fp64 stage
        ts = [h.host_time for h in r.history if h.stage == st]
        d = np.diff(ts)[1:] if len(ts) > 2 else np.array([np.nan])
        med.append(float(np.median(d)) * 1e3)
    if dist:
        t = torch.tensor(med, device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        med = t.tolist()
    del X0, Om
    torch.cuda.empty_cache()
    return {"workload": w["desc"] + ", mplobpcg-schol, "
                        f"{'row-sharded over ' + str(world) + ' GPUs' if shard else 'one GPU'}, "
                        f"capped at {iters}+{iters} iterations",
            "ms_per_iteration_fp32_stage": med[0], "ms_per_iteration_fp64_stage": med[1],
            "rows_per_gpu": n, "method": "median interval of the per-iteration records, max over ranks"}


def at_scale_kernels(mp, peak_gbs):
    """Per-kernel-family efficiency at the north-star target's per-GPU shape
    (256^3 rows / 8 GPUs = a 256 x 256 x 32 grid, k = 64, m = 80): a capped
    mixed-precision solve (8 iterations per stage) in profiling mode, algorithmic
    bytes / flops per family over its event-timed launches.  Evidence for the
    kernels' HBM / DMMA roofline at sizes where they are bandwidth- or
    compute-bound (cfg1's are latency-bound); not part of the timed metric."""
    import torch
    A = mp.laplace3d(256, 256, 32)
    cfg = mp.SolverConfig(k=64, block=80, tol=1e-10, maxit=8, variant="mplobpcg-schol")
    mp.solve(A, cfg, want_X=False, history=False)  # warm-up (allocations, attributes)
    torch.cuda.synchronize()
    with mp.profile():
        mp.solve(A, cfg, want_X=False, history=False)
        torch.cuda.synchronize()
        rep = mp.profile.report()
    out = {"workload": "3-D 7-pt Laplacian 256x256x32 (n=2.1M, the per-GPU rows of 256^3 on 8 GPUs), "
                       "k=64, m=80, mplobpcg-schol capped at 8+8 iterations, profiling pass",
           "hbm_peak_gbs": peak_gbs, "dmma_peak_tfs": DMMA_PEAK_TFS, "kernels": {}}
    for name, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
        if v["ms"] <= 0 or v["count"] == 0:
            continue
        gbs = v["bytes"] / (v["ms"] * 1e6) if v["bytes"] > 0 else None
        tfs = v["flops"] / (v["ms"] * 1e9) if v["flops"] > 0 else None
        out["kernels"][name] = {
            "launches": v["count"], "ms_per_launch": round(v["ms"] / v["count"], 4),
            "GBps": round(gbs, 1) if gbs else None,
            "hbm_frac": round(gbs / peak_gbs, 3) if gbs else None,
            "TFps": round(tfs, 2) if tfs else None,
            # fp64 families against the DMMA peak; the binary32 tensor-core families
            # (gram_f32 / gemm_f32: 8 bf16 part products each) against bf16 peak / 8
            "tensor_frac": (round(tfs / DMMA_PEAK_TFS, 3) if tfs and not name.endswith("_f32") else
                            round(8 * tfs / BF16_PEAK_TFS, 3) if tfs and name in TC_FAMILIES else None)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg1", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="mplobpcg-schol",
                    choices=["mplobpcg-schol", "dlobpcg-schol", "dlobpcg-dchol", "pinvit"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-at-scale", action="store_true",
                    help="skip the per-kernel efficiency pass at the 256^3 / 8-GPU per-rank shape")
    ap.add_argument("--shard", action="store_true",
                    help="at N = 1: the row-sharded code path over a 1-rank NCCL comm "
                         "(N > 1 is sharded by default)")
    ap.add_argument("--cfg4", action="store_true",
                    help="also time cfg4 (256^3, m = 80) per iteration at N = 1")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent single-GPU solves (weak scaling) instead of "
                         "one row-sharded solve")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
