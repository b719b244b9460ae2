"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import io
import sys
from collections import defaultdict

text = open(sys.argv[1]).read()
start = text.index('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
per = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = ("gemm" if "winograd_gemm" in name else "output_transform" if "output_transform" in name else
             "input_transform" if "input_transform" in name else "glue" if "requant" in name else
             "filter_transform" if "filter" in name else name[:60])
    v = float(r["Metric Value"])
    unit = r["Metric Unit"]
    unit = unit.strip().lower()
    v = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v  # -> usecond
    per[short][0] += 1
    per[short][1] += v
tot = sum(t for _, t in per.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} {n:8d} {t:12.1f} {t / tot * 100:6.1f}%")
