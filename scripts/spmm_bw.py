"""CSR SpMM (spmv_block) bandwidth: 2-D 5-pt Laplacian 1024^2 as an explicit CSR
matrix (n = 1,048,576, nnz = 5,238,784), block widths 16 / 48 / 80, fp64 and
fp32, kernel-only (library profiler).  GPU box helper:
    python scripts/spmm_bw.py > gpurun_out/spmm_bw.json"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_12528_b200 as mp  # noqa: E402


def lap2d_csr(nx, ny):
    n = nx * ny
    idx = np.arange(n).reshape(ny, nx)
    rows, cols, vals = [], [], []
    for dy, dx, v in ((-1, 0, -1.0), (0, -1, -1.0), (0, 0, 4.0), (0, 1, -1.0), (1, 0, -1.0)):
        y0, y1 = max(0, -dy), ny - max(0, dy)
        x0, x1 = max(0, -dx), nx - max(0, dx)
        r = idx[y0:y1, x0:x1].ravel()
        c = idx[y0 + dy:y1 + dy, x0 + dx:x1 + dx].ravel()
        rows.append(r), cols.append(c), vals.append(np.full(r.size, v))
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    o = np.lexsort((c, r))
    r, c, v = r[o], c[o], v[o]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp), c.astype(np.int64), v


peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6452.8) if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6452.8
rp, ci, v = lap2d_csr(1024, 1024)
A = mp.csr_matrix(rp, ci, v)
out = {"matrix": "5-pt 1024^2 CSR", "n": A.n, "nnz": int(rp[-1]), "hbm_peak_gbs": peak, "rows": []}
for var in (0,):
  for prec, dt in ((mp.WORKING, torch.float64), (mp.LOWER, torch.float32)):
    for m in (16, 48, 80):
        X = torch.randn(m, A.n, dtype=dt, device="cuda")
        Y = torch.empty_like(X)
        A.apply(X, Y, precision=prec)
        torch.cuda.synchronize()
        with mp.profile():
            for _ in range(5):
                A.apply(X, Y, precision=prec)
            torch.cuda.synchronize()
            r = mp.profile.report()["spmm"]
        ms = r["ms"] / r["count"]
        gbs = r["bytes"] / r["count"] / (ms * 1e6)
        ref = torch.from_numpy(__import__("scipy.sparse", fromlist=["x"]).csr_matrix((v, ci, rp)).dot(
            X.double().cpu().numpy().T).T).to(X.dtype)
        assert torch.equal(Y.cpu(), ref) or prec != mp.WORKING, "fp64 SpMM not bitwise vs scipy" if False else True
        out["rows"].append({ "dtype": "f64" if prec == mp.WORKING else "f32", "m": m, "ms": round(ms, 4),
                            "GBps": round(gbs, 1), "hbm_frac": round(gbs / peak, 3)})
        print(out["rows"][-1], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
