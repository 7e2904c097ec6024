"""Per-kernel SASS instruction counts of the in-tree libmpskq.so (evidence
that the overlap kernels issue DMMA / TMA bulk copies / FFMA64):

    python tools/sass_counts.py [> profiles/r02_sass_counts.json]

Runs `cuobjdump -sass` (no GPU needed) and counts, per function, the
mnemonics DMMA, DFMA, UBLKCP (cp.async.bulk), SYNCS (mbarrier), LDS, STG,
LDG and the total instruction count.
"""
import json
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2411_09336_b200" / "libmpskq.so"
KEYS = ("DMMA", "DFMA", "DMUL", "DADD", "UBLKCP", "SYNCS", "LDS", "LDG", "STG", "BAR", "SHFL")


def main():
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    counts = defaultdict(Counter)
    fn = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if fn and m:
            op = m.group(1)
            counts[fn]["total"] += 1
            for k in KEYS:
                if op == k or op.startswith(k):
                    counts[fn][k] += 1
    demangled = {}
    names = list(counts)
    try:
        dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
        demangled = dict(zip(names, dm))
    except OSError:
        pass
    rows = {demangled.get(k, k): dict(v) for k, v in sorted(counts.items()) if "kernel" in demangled.get(k, k)}
    json.dump({"library": str(LIB.name), "counts": rows}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
