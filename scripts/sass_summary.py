"""Per-kernel SASS opcode census of libmpeig_b200.so (cuobjdump -sass): proves which
kernels issue DMMA (fp64 mma.sync), UTC*MMA (tcgen05.mma), UTMALDG (TMA tensor loads),
LDGSTS (cp.async) and the TMEM loads, without a GPU.

    python scripts/sass_summary.py > profiles/r02_sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2302_12528_b200", "libmpeig_b200.so")
WATCH = ["DMMA", "HMMA", "UTCHMMA", "UTCQMMA", "UTCMMA", "UTCBAR", "UTMALDG", "UTMASTG",
         "LDTM", "STTM", "LDGSTS", "SYNCS", "DFMA", "FFMA"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                             text=True).stdout.split("\n")
        return out[:len(names)]
    except OSError:
        return names


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts, order = {}, []
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            order.append(cur)
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(1)
            for w in WATCH:
                if op == w:
                    counts[cur][w] += 1
    names = demangle(order)
    print("# cuobjdump -sass census of", os.path.relpath(LIB, ROOT), "(sm_100a)")
    print("# columns: opcode counts in the kernel's SASS (static, not dynamic)")
    print(f"# {'kernel':80s} " + " ".join(f"{w:>7s}" for w in WATCH))
    for raw, nm in sorted(zip(order, names), key=lambda t: t[1]):
        c = counts[raw]
        if not any(c[w] for w in WATCH):
            continue
        nm = re.sub(r"\(anonymous namespace\)::", "", nm)
        nm = re.sub(r"\(.*\)$", "", nm)
        print(f"{nm[:82]:82s} " + " ".join(f"{c[w]:7d}" for w in WATCH))


if __name__ == "__main__":
    main()
