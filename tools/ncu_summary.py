"""Summarise an ncu report: key throughput metrics, stall reasons, top SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
h, v = raw[0], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for k, x, u in zip(h, v, raw[1]):
    if k in want:
        print(f"{k:70s} {x} {u}")
stalls = [(k, x) for k, x in zip(h, v) if k.startswith("smsp__average_warps_issue_stalled") and
          k.endswith("_per_issue_active.ratio")]
stalls.sort(key=lambda t: -float(t[1] or 0))
print("-- stalls per issue")
for k, x in stalls[:8]:
    print(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {x}")
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
hdr, data = src[1], src[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
tot = sum(float(r[iS] or 0) for r in data)
print(f"-- top SASS by stall samples (total {tot:.0f})")
for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:ntop]:
    print(f"  {float(r[iS]) / tot * 100:5.1f}%  {r[iE]:>10s}  {r[1][:100]}")
