"""Key metrics of one or more ncu reports side by side: python tools/ncu_summary.py a.ncu-rep b.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Executed Instructions", "Issue Slots Busy", "Issued Warp Per Scheduler", "No Eligible",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Achieved Active Warps Per SM", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Memory Throughput", "DRAM Throughput", "Dynamic Shared Memory Per Block", "Local Memory Spilling Requests"]


def metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    d = {}
    for r in rows[1:]:
        x = dict(zip(hdr, r))
        d.setdefault(x.get("Metric Name"), (x.get("Metric Value"), x.get("Metric Unit")))
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        for k, u, v in zip(rr[0], rr[1], rr[2]):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                d["stall:" + k[len("smsp__pcsamp_warps_issue_stalled_"):]] = (v, u)
            if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"):
                d[k] = (v, u)
    return d


def main():
    ms = [metrics(p) for p in sys.argv[1:]]
    keys = KEYS + sorted({k for m in ms for k in m if k.startswith("stall:") or "." in k})
    for k in keys:
        vals = [m.get(k, ("-", ""))[0] for m in ms]
        if all(v == "-" for v in vals):
            continue
        print(f"{k:48s} " + " ".join(f"{v:>16s}" for v in vals) + "  " + (ms[0].get(k, ("", ""))[1] or ""))


if __name__ == "__main__":
    main()
