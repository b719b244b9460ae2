"""Per-SASS-line stall attribution of an ncu report: the top lines by samples
with their dominant stall reasons, plus region totals between markers.

usage: python tools/ncu_stalls.py rep.ncu-rep [ntop]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iS] or 0) for r in data)
agg = {h: 0.0 for _, h in reasons}
for r in data:
    for i, h in reasons:
        agg[h] += float(r[i] or 0)
print("total samples", tot)
print("by reason:", ", ".join(f"{h[6:]} {v / tot * 100:.1f}%" for h, v in sorted(agg.items(), key=lambda t: -t[1])[:10]))
for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:ntop]:
    top = sorted(((float(r[i] or 0), h[6:]) for i, h in reasons), reverse=True)[:3]
    print(f"{float(r[iS]) / tot * 100:5.1f}% {r[0][-5:]} {r[iE]:>9s}  {r[1][:60]:60s} " +
          " ".join(f"{h}:{v / max(1, float(r[iS])) * 100:.0f}%" for v, h in top if v > 0))
