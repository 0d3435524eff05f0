"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", name)
    name = name.replace("void ", "")
    name = re.sub(r"\(.*$", "", name)          # drop argument list
    base = re.sub(r"<.*$", "", name).strip()   # drop template args
    targs = re.search(r"<([^<>]*)>", name)
    return base + (f"<{targs.group(1)}>" if targs else "")


def main(path, out=None, title=""):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        k = short(r[ki])
        tot[k] += v
        cnt[k] += 1
    T = sum(tot.values())
    lines = [f"# {title}", f"# {'kernel':58s} launches   total_us  share  us/launch"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"{k:60s} {cnt[k]:6d} {v:10.1f} {v / T:6.3f} {v / cnt[k]:9.2f}")
    lines.append(f"# total {T:.1f} us over {sum(cnt.values())} launches")
    txt = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None,
         sys.argv[3] if len(sys.argv) > 3 else "")
