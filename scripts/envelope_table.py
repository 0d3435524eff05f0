"""Markdown table: the reference's per-stage iteration envelope under 1-ulp
start-block perturbations (tests/golden/envelope.json) next to the device's
counts on the same perturbed inputs (profiles/r02_envelope_device.json)."""
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
env = json.load(open(os.path.join(ROOT, "tests", "golden", "envelope.json")))
dev_p = os.path.join(ROOT, "profiles", "r02_envelope_device.json")
dev = json.load(open(dev_p)) if os.path.exists(dev_p) else {}


def fmt(a, st):
    x = a[:, st]
    if x.max() == 0:
        return "-"
    return f"{int(x.min())}-{int(x.max())} ({x.mean():.0f} +- {x.std(ddof=1):.0f})"


print("| case | reference (p=0) | reference stage 1: range (mean +- sd) | stage 2 | device (p=0) | device stage 1 mean | stage 2 mean |")
print("|---|---|---|---|---|---|---|")
for c in sorted(env):
    e = env[c]
    a = np.array([e["ref"]] + e["perturbed"], float)
    d = dev.get(c)
    dv = d["device_unperturbed"] if d else None
    dm = np.array(d["device_perturbed"], float).mean(0) if d else None
    print(f"| {c} | {e['ref'][0]}+{e['ref'][1]} | {fmt(a, 0)} | {fmt(a, 1)} | "
          f"{(str(dv[0]) + '+' + str(dv[1])) if dv else 'n/a'} | "
          f"{('%.1f' % dm[0]) if d and dm[0] > 0 else '-'} | {('%.1f' % dm[1]) if d else 'n/a'} |")
