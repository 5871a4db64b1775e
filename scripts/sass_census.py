#!/usr/bin/env python3
"""Per-kernel SASS census of libelis.so (cuobjdump -sass): the Blackwell instructions that show
which hardware path each kernel takes -- tcgen05 MMAs (UTCHMMA: kind::f16 / tf32, UTCQMMA:
kind::f8f6f4; .2CTA = cta_group::2), TMA (UTMALDG load, UTMASTG store, UBLKCP bulk copy), TMEM
(LDTM / STTM), mbarrier (SYNCS), MUFU and the fp32x2 FFMA2 / FADD2.

    python scripts/sass_census.py [paper_2505_09142_b200/libelis.so] > profiles/rNN_sass_census.md
"""
from __future__ import annotations

import re
import subprocess
import sys
from collections import Counter, defaultdict

OPS = ["UTCHMMA", "UTCQMMA", "UTCMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "SYNCS", "MUFU.EX2",
       "FFMA2", "FADD2", "HMMA", "LDSM", "STL", "LDL"]


def demangle(name: str) -> str:
    try:
        out = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        return name
    out = re.sub(r"elis::\(anonymous namespace\)::|elis::<unnamed>::", "", out)
    out = re.sub(r"\(.*\)$", "", out)
    return out


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2505_09142_b200/libelis.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    counts: dict[str, Counter] = defaultdict(Counter)
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = demangle(m.group(1))
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        op = m.group(1)
        for key in OPS:
            if op == key or op.startswith(key + "."):
                counts[cur][key + (".2CTA" if key.startswith("UTC") and ".2CTA" in op else "")] += 1
                break
    cols = sorted({c for v in counts.values() for c in v}, key=lambda c: (OPS.index(c.split(".2CTA")[0]) if c.split(".2CTA")[0] in OPS else 99, c))
    print(f"# SASS census of {lib} (static instruction counts per kernel; cuobjdump -sass)\n")
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    for k in sorted(counts):
        if not any(counts[k].values()):
            continue
        print(f"| `{k}` | " + " | ".join(str(counts[k].get(c, "")) for c in cols) + " |")


if __name__ == "__main__":
    main()
