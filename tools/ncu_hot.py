#!/usr/bin/env python
"""Top SASS instructions of an ncu report by warp-stall samples.
Usage: python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main(rep, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    samp = [h for h in hdr if h.startswith("Warp Stall Sampling (All")]
    key = samp[0] if samp else None
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    recs = []
    for r in rows[2:]:
        try:
            tot = int(r[idx[key]] or 0)
        except (ValueError, TypeError):
            continue
        top = sorted(((int(r[idx[h]] or 0), h) for h in stall_cols), reverse=True)[:2]
        recs.append((tot, r[idx["Address"]] if "Address" in idx else "", r[idx["Source"]], top))
    total = sum(x[0] for x in recs)
    for tot, addr, src, top in sorted(recs, reverse=True)[:n]:
        print(f"{tot:6d} {tot / total:5.1%} {addr:>6s} {src[:70]:70s} {top}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
