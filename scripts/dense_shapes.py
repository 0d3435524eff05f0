"""Gram / block-GEMM throughput at the solver's shapes (GPU box helper):

    python scripts/dense_shapes.py [n] > gpurun_out/dense_shapes.json

Times the library kernels through the C ABI (mpeig_gram_* / mpeig_gemm_*),
kernel-only via the library's CUDA-event profiler, for the shapes one LOBPCG
iteration issues at m = 16 / 48 / 80 (project-out Grams [X P]^T W, CholQR
Grams W^T W, S^T AS, the S C / AS C update, W - B G, V U^-1)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2302_12528_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 * 1024 * 1024
ms_list = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 48, 80]
dtypes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["f64", "f32"]
reps = 5
ctx = mp.default_context()
# MPEIG_OPTS="gemm_tma2=2,gram_tma=0": process options (kernel-selection experiments)
for kv in filter(None, os.environ.get("MPEIG_OPTS", "").split(",")):
    key, val = kv.split("=")
    assert ctx.lib.mpeig_set_process_option(key.encode(), int(val)) == 0, kv
out = {"n": n, "rows": []}


def prof(fn):
    fn()
    torch.cuda.synchronize()
    with mp.profile():
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        rep = mp.profile.report()
    return rep


for sfx in dtypes:
    dt = torch.float64 if sfx == "f64" else torch.float32
    ld = n
    for m in ms_list:
        s = 3 * m
        S = torch.randn(s, ld, dtype=dt, device="cuda")  # column-major n x s (ld = n)
        G = torch.zeros(s, s, dtype=dt, device="cuda")
        Cm = torch.randn(s, s, dtype=dt, device="cuda")
        Y = torch.empty(2 * m, ld, dtype=dt, device="cuda")
        p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        gram = getattr(ctx.lib, f"mpeig_gram_{sfx}")
        gemm = getattr(ctx.lib, f"mpeig_gemm_{sfx}")
        cases = [
            ("gram S^T S", s, s, lambda: gram(ctx.h, n, s, p(S), ld, s, p(S), ld, p(G))),
            ("gram [X P]^T W", 2 * m, m, lambda: gram(ctx.h, n, 2 * m, p(S), ld, m, p(S[2 * m:]), ld, p(G))),
            ("gram W^T W", m, m, lambda: gram(ctx.h, n, m, p(S[2 * m:]), ld, m, p(S[2 * m:]), ld, p(G))),
        ]
        for name, ka, kb, fn in cases:
            ctx.check(fn())
            r = prof(lambda: ctx.check(fn()))["gram" if sfx == "f64" else "gram_f32"]
            ms = r["ms"] / r["count"]
            out["rows"].append({"dtype": sfx, "m": m, "op": name, "shape": [ka, kb],
                                "ms": round(ms, 4), "TFps": round(2.0 * n * ka * kb / (ms * 1e9), 2),
                                "GBps": round(r["bytes"] / r["count"] / (ms * 1e6), 1)})
        one = 1.0
        gcases = [
            ("gemm S C (-> X, P)", s, 2 * m, lambda: gemm(ctx.h, n, s, 2 * m, one, p(S), ld, p(Cm), s, 0.0, None, 0, p(Y), ld)),
            ("gemm W - B G", 2 * m, m, lambda: gemm(ctx.h, n, 2 * m, m, -one, p(S), ld, p(Cm), s, one, p(Y), ld, p(Y), ld)),
            ("gemm V U^-1", m, m, lambda: gemm(ctx.h, n, m, m, one, p(S), ld, p(Cm), s, 0.0, None, 0, p(Y), ld)),
        ]
        for name, k, c, fn in gcases:
            ctx.check(fn())
            r = prof(lambda: ctx.check(fn()))["gemm" if sfx == "f64" else "gemm_f32"]
            ms = r["ms"] / r["count"]
            out["rows"].append({"dtype": sfx, "m": m, "op": name, "shape": [k, c],
                                "ms": round(ms, 4), "TFps": round(2.0 * n * k * c / (ms * 1e9), 2),
                                "GBps": round(r["bytes"] / r["count"] / (ms * 1e6), 1)})
        del S, G, Cm, Y
        torch.cuda.empty_cache()
for r in out["rows"]:
    print(r, file=sys.stderr)
print(json.dumps(out, indent=1))
