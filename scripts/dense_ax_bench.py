"""cfg3 dense operator apply A·X (n = 16384, m = 96, fp64): the library's DMMA
block GEMM (k_gemm_dmma via mpeig_gemm_f64, K = n) against cuBLAS DGEMM (the
dense operator's current apply), CUDA events on the launching stream.

    python scripts/dense_ax_bench.py [n] [m]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2302_12528_b200 as mp  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 96
    ctx = mp.default_context()
    out = {"n": n, "m": m}
    for dt in (torch.float64, torch.float32):
        g = torch.Generator(device="cuda").manual_seed(0)
        A = torch.randn((n, n), dtype=dt, device="cuda", generator=g)  # column-major = A^T rows
        X = torch.randn((m, n), dtype=dt, device="cuda", generator=g)
        Y1 = torch.empty((m, n), dtype=dt, device="cuda")
        Y2 = torch.empty((m, n), dtype=dt, device="cuda")
        flops = 2.0 * n * n * m
        bytes_ = A.element_size() * (n * n + 2 * n * m)
        f = ctx.lib.mpeig_gemm_f64 if dt == torch.float64 else ctx.lib.mpeig_gemm_f32

        def ours():
            ctx.check(f(ctx.h, n, n, m, 1.0, C.c_void_p(A.data_ptr()), n, C.c_void_p(X.data_ptr()), n,
                        0.0, None, n, C.c_void_p(Y1.data_ptr()), n))

        def cublas():
            # column-major Y (n x m) = A (n x n) X (n x m)  <=>  row-major Y^T = X^T A^T
            torch.matmul(X, A, out=Y2)

        sfx = "f64" if dt == torch.float64 else "f32"
        for name, fn in ((f"ours_{sfx}", ours), (f"cublas_{sfx}", cublas)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            with mp.profile():
                fn()
                torch.cuda.synchronize()
                rep = mp.profile.report()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                fn()
            torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            key = "gemm" if "gemm" in rep else "gemm_f32"
            if name.startswith("ours") and key in rep:
                ms = rep[key]["ms"] / rep[key]["count"]  # kernel-only (library events)
            out[name] = {"ms": round(ms, 4), "TFps": round(flops / ms / 1e9, 2),
                         "GBps": round(bytes_ / ms / 1e6, 1)}
        out[f"max_rel_diff_{sfx}"] = (Y1.double() - Y2.double()).abs().max().item() / Y2.double().abs().max().item()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
