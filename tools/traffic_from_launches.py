#!/usr/bin/env python
"""Per-pass DRAM traffic of the node-update kernels from an ncu launch list (tools/profile_cfg3.sh)
-> profiles/ncu_traffic.json[key], read by bench.py for roofline.traffic.
Usage: python tools/traffic_from_launches.py launches.csv KEY PASSES
KEY = "<config>:<precision>:<layout>:<form>:<nv>" (bench.py's lookup key)."""
import collections
import csv
import json
import os
import sys

NODE_KERNELS = ("tile_update", "side_rows", "warp_update", "hub_fast_update", "node_update", "hub_update")


def main(path, key, passes):
    hdr = None
    byk = collections.defaultdict(float)
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        if not any(k in name for k in NODE_KERNELS):
            continue
        if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            byk[name[:name.find("(")]] += float(d["Metric Value"].replace(",", ""))
    per_pass = sum(byk.values()) / passes
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[key] = per_pass
    data.setdefault("_source", {})[key] = {
        "launch_list": os.path.basename(path), "passes": passes,
        "bytes_per_pass_by_kernel": {k: v / passes for k, v in byk.items()},
        "note": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, cold cache, serialised"}
    json.dump(data, open(out, "w"), indent=1, sort_keys=True)
    print(key, per_pass)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]))
