#!/usr/bin/env python
"""Summarise an ncu report (first kernel): key throughput / stall numbers as JSON.
Usage: python tools/ncu_summary.py report.ncu-rep [--source]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main():
    rep = sys.argv[1]
    r = raw(rep)
    res = {"kernel": r.get("Kernel Name", ("?", ""))[0]}
    for k in KEYS:
        if k in r:
            res[k] = f"{r[k][0]} {r[k][1]}".strip()
    if "--source" in sys.argv:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr = rows[1]
        idx = {h: i for i, h in enumerate(hdr)}
        stalls = {h: 0 for h in hdr if h.startswith("stall_") and "Not Issued" not in h}
        for row in rows[2:]:
            for h in stalls:
                try:
                    stalls[h] += int(row[idx[h]] or 0)
                except ValueError:
                    pass
        res["stall_samples"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:8])
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
