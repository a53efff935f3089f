#!/usr/bin/env python3
"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

    python tools/ncu_summary.py full  <report.ncu-rep> <out.json> [--algo-bytes B]
    python tools/ncu_summary.py launches <launches.csv> <out.json>
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_write.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "dram__cycles_active.min.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.max.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_op_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
]

UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "byte": 1, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def full(rep, out, algo):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    kern = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    d[k] = float(v) * UNIT.get(units[i], 1.0) if units[i] in UNIT else float(v)
                    d[k + ".unit"] = "SI (bytes / s)" if units[i] in UNIT else units[i]
                except ValueError:
                    d[k] = v
        kern.append(d)
    k0 = kern[0]
    res = {"source": rep, "kernels": kern,
           "dram_bytes_per_launch": k0.get("dram__bytes_read.sum", 0) + k0.get("dram__bytes_write.sum", 0),
           "algorithmic_bytes_per_launch": algo}
    if algo and isinstance(k0.get("smsp__inst_executed.sum"), float):
        # thread-instructions per number = warp-instructions x 32 / (n x T),
        # n x T = algorithmic bytes / 8
        res["thread_instructions_per_number"] = k0["smsp__inst_executed.sum"] * 32 / (algo / 8)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}))


def launches(path, out):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    per = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", "")) * (1e3 if r["Metric Unit"] == "us" else 1e6 if r["Metric Unit"] == "ms" else 1)
        per.setdefault(r["Kernel Name"], []).append(ns)
    tot = sum(sum(v) for v in per.values())
    res = {"source": path, "total_ns": tot,
           "kernels": {k: {"launches": len(v), "total_ns": sum(v), "mean_ns": sum(v) / len(v), "share": sum(v) / tot}
                       for k, v in per.items()}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    algo = float(sys.argv[sys.argv.index("--algo-bytes") + 1]) if "--algo-bytes" in sys.argv else None
    full(src, dst, algo) if mode == "full" else launches(src, dst)
