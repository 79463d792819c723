"""Form A to convergence (move_tol 1e-6, cap 1000) on a 1M-node mesh: per-pass graph vs the
dataflow launch (rounds of 64 passes, replay of the stopping round).  usage: python tools/conv_probe.py"""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1502_00355_b200 as ts  # noqa: E402
from paper_1502_00355_b200 import capi  # noqa: E402

xy, tri = ts.delaunay_arrays(1_000_000, 42)
ctx = capi.Context(0)
dm = capi.DeviceMesh(ctx, xy, tri, None, order=ctx.hilbert_order(xy))
cfg = capi.make_cfg(form="a", max_iters=1000, move_tol=1e-6, bbox_diag=ts.bbox_diagonal(xy))
for rep in range(2):
    for flow in ("0", "1"):
        os.environ["TSG_FORMA_FLOW"] = flow
        dm.restore_coords()
        r = dm.smooth(cfg)
        print("flow", flow, "iterations", r["iterations"], r["stop"], "device ms", round(r["device_ms"], 2),
              "schedule", r["schedule"], flush=True)
