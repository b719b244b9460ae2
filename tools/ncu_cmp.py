"""Compare selected raw metrics (and the top warp-stall reasons) of ncu reports.

usage: python tools/ncu_cmp.py a.ncu-rep [b.ncu-rep ...] [--kernel REGEX]
"""
import csv, io, re, subprocess, sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
kre = None
if "--kernel" in sys.argv:
    kre = re.compile(sys.argv[sys.argv.index("--kernel") + 1])
    args = [a for a in args if a != sys.argv[sys.argv.index("--kernel") + 1]]
BASE = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size"]
for rep in args:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for row in rows[2:]:
        name = row[h.index("Kernel Name")]
        if kre and not kre.search(name):
            continue
        print(rep, name[:70])
        for m in BASE:
            if m in h:
                print(f"   {m:60s} {row[h.index(m)]}")
        stalls = []
        for i, m in enumerate(h):
            mm = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", m)
            if mm:
                try:
                    stalls.append((float(row[i]), mm.group(1)))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("   stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))
