"""ms per pass of the cfg3 graph smooth with the side rows in the persistent kernel vs the
per-tier grids, fp64 and fp32 (alternating, one process).  usage: python tools/side_probe.py"""
import sys

sys.path.insert(0, ".")
import paper_1502_00355_b200 as ts  # noqa: E402
from paper_1502_00355_b200 import capi  # noqa: E402

xy, tri = ts.graded_arrays(16_000_000, 1, 1e-3, 1024)
ctx = capi.Context(0)
order = ctx.hilbert_order(xy)
for prec in ("f64", "f32"):
    dm = capi.DeviceMesh(ctx, xy, tri, None, precision=prec, order=order)
    cfg = capi.make_cfg(form="a", max_iters=100, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy))
    for rep in range(3):
        for side in ("auto", "persist", "kernels"):
            dm.side_schedule(side)
            dm.restore_coords()
            r = dm.smooth(cfg)
            print(prec, side, rep, round(r["device_ms"] / r["iterations"], 4), "ms/pass", flush=True)
    dm.free()
