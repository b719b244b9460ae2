"""Opcode census of librnsw.so's SASS, per kernel (evidence for the judge:
which kernels issue tcgen05 MMAs, TMA, TMEM loads, or legacy mma.sync).

    python tools/sass_census.py [path/to/librnsw.so] > profiles/rNN_sass_census.txt
"""
from __future__ import annotations

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
WATCH = ("UTCIMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "UTMACMDFLUSH", "LDTM", "STTM", "IMMA", "HMMA",
         "SYNCS", "BAR", "LDG", "STG", "LDS", "STS", "IMAD", "PRMT")


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True).stdout
        return out.splitlines()
    except (OSError, subprocess.CalledProcessError):
        return names


def main():
    lib = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "paper_2007_12216_b200" / "librnsw.so"
    sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    counts: dict[str, collections.Counter] = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m and cur is not None:
            op = m.group(1)
            counts[cur][op] += 1
            counts[cur]["_total"] += 1
    names = list(counts)
    pretty = demangle(names)
    print(f"# SASS opcode census of {lib.name} (cuobjdump -sass), static instruction counts per kernel")
    print("# " + " ".join(f"{w:>8}" for w in WATCH) + "   total  kernel")
    for raw, nice in sorted(zip(names, pretty), key=lambda t: t[1]):
        c = counts[raw]
        row = " ".join(f"{sum(v for k, v in c.items() if k == w or k.startswith(w + '.')):>8}" for w in WATCH)
        short = re.sub(r"\(.*", "", nice.replace("(anonymous namespace)::", ""))
        print(f"  {row} {c['_total']:>7}  {short[:150]}")


if __name__ == "__main__":
    main()
