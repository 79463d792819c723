#!/usr/bin/env python
"""Aggregate an ncu --csv launch list (gpu__time_duration / dram bytes per launch) by kernel.
The pass kernels (the smoothing step) are listed first with their share of the step; mesh prep
and the reorder kernels follow with their share of everything listed.
Usage: python tools/launches.py launches.csv"""
import collections
import csv
import sys


def main(path):
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"]
        k = k[:k.find("(")] if "(" in k else k
        m, v = d["Metric Name"], float(d["Metric Value"].replace(",", ""))
        a = agg[k]
        if m == "gpu__time_duration.sum":
            a[0] += 1
            a[1] += v
        elif m == "dram__bytes_read.sum":
            a[2] += v
        elif m == "dram__bytes_write.sum":
            a[3] += v
    step = {k: a for k, a in agg.items() if any(p in k for p in PASS_KERNELS)}
    rest = {k: a for k, a in agg.items() if k not in step}
    for title, group in (("pass kernels (share of the smoothing step)", step),
                         ("mesh prep / reorder (share of these)", rest)):
        if not group:
            continue
        tot = sum(a[1] for a in group.values())
        print(f"# {title}")
        print(f"{'kernel':58s} {'n':>4s} {'us/launch':>10s} {'share':>6s} {'MB rd/l':>9s} {'MB wr/l':>9s}")
        for k, a in sorted(group.items(), key=lambda x: -x[1][1]):
            n = max(1, a[0])
            print(f"{k[-58:]:58s} {a[0]:4d} {a[1] / n / 1e3:10.1f} {a[1] / tot:6.1%} {a[2] / n / 1e6:9.1f} "
                  f"{a[3] / n / 1e6:9.1f}")


PASS_KERNELS = ("tile_update", "tile_flow", "side_rows", "warp_update", "hub_fast_update", "hub_update",
                "node_update", "formb_", "finalize_pass", "flow_reset", "reset_pass_state", "peer_")


if __name__ == "__main__":
    main(sys.argv[1])
