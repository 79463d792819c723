#!/usr/bin/env python
"""Variant sweep on one mesh (layout x precision x strategy x form x swap): one JSON line per
variant with node-updates/s of the graph-driven pass loop and the node-kernel time per pass.
Used to justify the default configuration — not the headline bench."""
import argparse
import itertools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--nodes", type=int, default=None)
    ap.add_argument("--passes", type=int, default=100)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--layouts", default="aos,soa")
    ap.add_argument("--precisions", default="f64,f32")
    ap.add_argument("--strategies", default="fused,twophase")
    ap.add_argument("--forms", default="a")
    ap.add_argument("--swaps", default="pingpong")
    ap.add_argument("--chunks", type=int, default=1)
    ap.add_argument("--reorder", default="1")
    args = ap.parse_args()
    import paper_1502_00355_b200 as ts
    from paper_1502_00355_b200 import capi

    cfg = dict(bench.CONFIGS[args.config])
    xy, tri, _ = bench.make_mesh(ts, cfg, args.nodes)
    nv, nt = len(xy), len(tri)
    topo = ts.topology(nv, tri)
    sum_deg = int(topo["nbr_off"][-1])
    diag = ts.bbox_diagonal(xy)
    ctx = capi.Context(0)
    peak, _ = bench.measured_peak()
    for layout, prec, strat, form, swap, reorder in itertools.product(
            args.layouts.split(","), args.precisions.split(","), args.strategies.split(","),
            args.forms.split(","), args.swaps.split(","), [int(x) for x in args.reorder.split(",")]):
        order = capi.hilbert_order(xy) if reorder else None
        t0 = time.time()
        dm = capi.DeviceMesh(ctx, xy, tri, topo, layout=layout, precision=prec, order=order)
        up = time.time() - t0
        mk = lambda drv: capi.make_cfg(form=form, strategy=strat, chunks=args.chunks, swap=swap,
                                       max_iters=args.passes, driver=drv, move_tol=0.0, bbox_diag=diag)
        dm.restore_coords()
        dm.smooth(mk("graph"))
        tot, its = 0.0, 0
        for _ in range(args.steps):
            dm.restore_coords()
            r = dm.smooth(mk("graph"))
            tot += r["device_ms"]
            its += r["iterations"]
        dm.restore_coords()
        rs = dm.smooth(mk("stream"))
        node_ms = rs["node_kernel_ms"] / max(1, rs["iterations"])
        b = bench.algorithmic_bytes_per_pass(nv, nt, sum_deg, prec)
        out = dict(config=args.config, nv=nv, layout=layout, precision=prec, strategy=strat, form=form, swap=swap,
                   chunks=args.chunks, reorder=reorder, node_updates_per_s=nv * its / (tot / 1000.0),
                   ms_per_pass=tot / its, node_kernel_ms=node_ms, roofline_frac=b / (node_ms / 1000) / 1e9 / peak,
                   accepted_first=int(rs["accepted"][0]), upload_s=up, device_gb=dm.device_bytes / 1e9)
        print(json.dumps(out), flush=True)
        dm.free()


if __name__ == "__main__":
    main()
