"""Small smooths for compute-sanitizer, checked against the oracle: Form A through the dataflow
launch (tile_flow) and the per-pass kernels, the side-row kernels, Form B schedules, device
topology / layout / quality audit.  Usage:
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_flow.py
SAN_FORMB selects the Form B schedules (default flow,chunks,levels).  synccheck reports the
level barrier of formb_chunk_update (an unconditional __syncthreads that every thread executes,
reached by warps that are not reconverged after the per-lane level work); run it separately.
SAN_DRIVERS=stream limits the per-pass runs to plain launches (racecheck does not follow kernel
boundaries inside conditional-WHILE graph bodies: it reports the first shared-memory write of a
CTA against the previous launch's CTA, and can crash on them)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1502_00355_b200 as ts  # noqa: E402
from paper_1502_00355_b200 import capi  # noqa: E402
from oracle import Port  # noqa: E402  (the checker)

ctx = capi.Context(0)
port = Port()
xy, tri = ts.delaunay_arrays(6000, 3)
topo = ts.topology(len(xy), tri)
want = port.smooth(xy, tri, form="a", max_iters=4, move_tol=0.0)
for layout in ("aos", "soa"):
    dm = capi.DeviceMesh(ctx, xy, tri, topo, layout=layout, order=capi.hilbert_order(xy))
    for driver in ("graph", "stream"):
        dm.set_coords(xy)
        r = dm.smooth(capi.make_cfg(form="a", max_iters=4, move_tol=0.0, driver=driver))
        assert np.array_equal(dm.get_coords().view(np.uint64), want.xy.view(np.uint64)), (layout, driver)
        print(layout, driver, r["schedule"], "ok")
    dm.free()
print("sanitize_flow: OK")

# Side rows (valence >= 32: persistent side_rows and the per-tier grids), Form B schedules,
# device topology / layout / quality audit.
xy, tri = ts.graded_arrays(12000, 3, 4e-3, 300)
topo = ctx.topology(len(xy), tri)
assert ctx.layout_check(xy, tri, topo, ctx.hilbert_order(xy)) == ""
want = port.smooth(xy, tri, form="a", max_iters=3, move_tol=0.0)
dm = capi.DeviceMesh(ctx, xy, tri, topo, order=capi.hilbert_order(xy))
DRIVERS = os.environ.get("SAN_DRIVERS", "graph,stream").split(",")
for side in ("persist", "kernels"):
    dm.side_schedule(side)
    for driver in DRIVERS:
        dm.set_coords(xy)
        dm.smooth(capi.make_cfg(form="a", max_iters=3, move_tol=0.0, driver=driver))
        assert np.array_equal(dm.get_coords().view(np.uint64), want.xy.view(np.uint64)), (side, driver)
        print("side", side, driver, "ok")
fin = want.xy
assert np.array_equal(dm.tri_alpha(), np.array([port.alpha(tuple(fin[a]), tuple(fin[b]), tuple(fin[c]))
                                                for a, b, c in tri]))
dm.free()
for chunks in (1, 8):
    want = port.smooth(xy, tri, form="b", chunks=chunks, max_iters=3, move_tol=0.0)
    dm = capi.DeviceMesh(ctx, xy, tri, topo)
    for sched in os.environ.get("SAN_FORMB", "flow,chunks,levels").split(","):
        dm.formb_schedule(sched)
        dm.set_coords(xy)
        for driver in DRIVERS:
            dm.set_coords(xy)
            dm.smooth(capi.make_cfg(form="b", chunks=chunks, max_iters=3, move_tol=0.0, driver=driver))
            assert np.array_equal(dm.get_coords().view(np.uint64), want.xy.view(np.uint64)), (chunks, sched)
            print("form b", chunks, sched, driver, "ok")
    dm.free()
print("sanitize_flow: side rows, Form B, prep OK")
