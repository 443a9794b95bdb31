#!/usr/bin/env python
"""Summarise an .ncu-rep: key throughput metrics, stall reasons by code region, top stalled SASS."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15

def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "sm__cycles_active.avg"]
for n, uu, vv in zip(h, u, v):
    if n in want:
        print(f"{n} = {vv} {uu}")
stall = {n: vv for n, vv in zip(h, v) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
tot = sum(float(x.replace(",", "") or 0) for x in stall.values())
print("stall samples:", {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(float(x.replace(",", "")) / tot * 100, 1)
                         for k, x in sorted(stall.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]})
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
hh = src[1]
rows = [dict(zip(hh, x)) for x in src[2:] if len(x) == len(hh)]
rows.sort(key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))
print("top stalled SASS:")
for x in rows[:top]:
    print(" ", x["Warp Stall Sampling (All Samples)"], x["Instructions Executed"], x["Address"][-5:], x["Source"].strip()[:70])
