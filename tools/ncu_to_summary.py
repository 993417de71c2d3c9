"""ncu --set full reports -> profiles/<round>/ncu_<tag>_summary.json (read by bench.py for roofline.traffic) and
the details pages as CSV.

  python tools/ncu_to_summary.py <out_dir> <tag> <config> <kernel>=<report.ncu-rep> [...]
"""
import csv
import io
import json
import os
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "smsp__thread_inst_executed_per_inst_executed.ratio", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__inst_executed.sum"]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    out_dir, tag, cfg = sys.argv[1:4]
    summary = {cfg: {}, "how": "ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 1 -c 1 "
                                "python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline (1 x B200)"}
    for arg in sys.argv[4:]:
        kernel, rep = arg.split("=", 1)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        names, units, vals = rows[0], rows[1], rows[2]
        d = dict(zip(names, zip(vals, units)))
        rb = float(d["dram__bytes_read.sum"][0].replace(",", "")) * UNIT.get(d["dram__bytes_read.sum"][1], 1.0)
        wb = float(d["dram__bytes_write.sum"][0].replace(",", "")) * UNIT.get(d["dram__bytes_write.sum"][1], 1.0)
        k = {"dram_read_bytes": rb, "dram_write_bytes": wb, "traffic_bytes": rb + wb}
        for m in RAW:
            if m in d:
                k[m] = f"{d[m][0]} {d[m][1]}"
        summary[cfg][kernel] = k
        det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        with open(os.path.join(out_dir, f"{kernel}_{tag}_details.csv"), "w") as f:
            f.write(det)
    with open(os.path.join(out_dir, f"ncu_{tag}_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
