"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv): per kernel kind, launches, device time, share and DRAM bytes.

usage: python tools/launch_summary.py launches.csv [--traffic-json OUT --shard B]
  --traffic-json writes {"<kind>:b<B>": dram bytes summed over that kind's launches}
  (the bench's roofline.traffic for the same per-step launch set).
"""
import csv
import io
import json
import sys
from collections import defaultdict

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
        "byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}


def kind_of(name: str) -> str:
    for key, kind in (("winograd_gemm", "gemm"), ("output_transform", "output_transform"), ("output_umma", "output_transform"),
                      ("output_kron", "output_transform"), ("input_umma", "input_transform"),
                      ("input_transform", "input_transform"), ("smallc_product", "product"),
                      ("requant", "glue"), ("filter_transform", "filter_transform (setup, not in the step)")):
        if key in name:
            return kind
    return name[:60]


text = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
launch = defaultdict(dict)
for r in rows:
    try:
        val = float(r["Metric Value"].replace(",", ""))
    except ValueError:  # "n/a" (e.g. a DRAM counter ncu could not collect for a launch)
        continue
    launch[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = val * UNIT.get(r["Metric Unit"].strip().lower(), 1.0)
per = defaultdict(lambda: [0, 0.0, 0.0])
for (lid, name), m in launch.items():
    k = kind_of(name)
    per[k][0] += 1
    per[k][1] += m.get("gpu__time_duration.sum", 0.0)
    per[k][2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
step = {k: v for k, v in per.items() if "setup" not in k}
tot = sum(v[1] for v in step.values())
print(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'share':>7s} {'dram_GB':>9s} {'GB/s':>7s}")
for k, (n, t, b) in sorted(per.items(), key=lambda kv: -kv[1][1]):
    share = f"{t / tot * 100:6.1f}%" if k in step else "     - "
    print(f"{k:44s} {n:8d} {t:10.1f} {share} {b / 1e9:9.3f} {b / t / 1e3 if t else 0:7.0f}")
if "--traffic-json" in sys.argv:
    out = sys.argv[sys.argv.index("--traffic-json") + 1]
    shard = sys.argv[sys.argv.index("--shard") + 1]
    json.dump({f"{k}:b{shard}": round(v[2]) for k, v in step.items()}, open(out, "w"), indent=1)
    print("wrote", out)
