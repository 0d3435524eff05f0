"""Device iteration counts on the reference envelope's perturbed start blocks
(tests/golden/make_envelope.py), next to the reference's.  GPU box helper:

    python scripts/envelope_device.py [case ...] > gpurun_out/envelope_device.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2302_12528_b200 as mp  # noqa: E402
from test_gpu_solver import device_perturbed_runs, envelope  # noqa: E402

cases = sys.argv[1:] or ["lap3d8-dlobpcg-dchol", "lap3d8-dlobpcg-schol", "lap3d8-mplobpcg-schol",
                         "lap3d16-dlobpcg-dchol", "lap3d16-dlobpcg-schol", "lap3d16-mplobpcg-schol",
                         "lap2d50-mplobpcg-schol", "dense256-dlobpcg-dchol", "dense256-mplobpcg-schol",
                         "lap2d5x500-mplobpcg-schol", "cfg1-mplobpcg-schol", "cfg1-dlobpcg-dchol",
                         "cfg1-dlobpcg-schol", "lap2d64k32-dlobpcg-dchol", "lap2d64k32-mplobpcg-schol",
                         "lap2d128k32-dlobpcg-dchol", "ks32-dlobpcg-dchol", "ks32-mplobpcg-schol"]
out = {}
for c in cases:
    env = envelope(c)
    npert = env["npert"] if env else 16
    runs = device_perturbed_runs(mp, c, npert)
    d = np.array(runs[1:], float)
    row = {"device_unperturbed": list(runs[0]), "device_perturbed": [list(r) for r in runs[1:]],
           "device_mean": d.mean(0).tolist()}
    if env:
        a = np.array(env["perturbed"], float)
        row.update(reference=env["ref"], reference_mean=a.mean(0).tolist(),
                   reference_min=a.min(0).tolist(), reference_max=a.max(0).tolist())
    out[c] = row
    print(c, json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
