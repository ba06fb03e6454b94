#!/usr/bin/env python
"""Per-kernel histogram of the Blackwell-specific SASS instructions in libams.so (proof of
tcgen05 / TMEM / TMA use):  python scripts/sass_histogram.py > profiles/sass_<round>.txt

Counts, per kernel instantiation: UTC*MMA (tcgen05.mma: HMMA = f16/bf16, IMMA = i8),
UTCBAR (tcgen05.commit), LDTM (tcgen05.ld), UTMALDG (TMA tensor loads), UBLKCP (bulk
copies), LDGSTS (cp.async), UTMACCTL (tensor-map prefetch), plus the total instruction
count.  The library's build id (ams_build_id: sources + flags) heads the file."""
import collections
import hashlib
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2508_10259_b200", "libams.so")
OPS = ("UTCHMMA", "UTCIMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "LDGSTS", "UTMACCTL")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return out if len(out) == len(names) else names


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts, total, order = {}, collections.Counter(), []
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            order.append(cur)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            op = m.group(1)
            total[cur] += 1
            for o in OPS:
                if op.startswith(o):
                    counts[cur][o] += 1
    sys.path.insert(0, ROOT)
    import paper_2508_10259_b200 as ams
    print(f"# libams.so ams_build_id {ams.ams_build_id()}")
    print(f"# {'kernel':<100s} " + " ".join(f"{o:>8s}" for o in OPS) + f" {'instr':>8s}")
    names = demangle(order)
    for n, dn in sorted(zip(order, names), key=lambda t: t[1]):
        short = re.sub(r"\(.*", "", dn.replace("(anonymous namespace)::", ""))
        print(f"  {short[:100]:<100s} " + " ".join(f"{counts[n][o]:8d}" for o in OPS) + f" {total[n]:8d}")


if __name__ == "__main__":
    sys.exit(main())
