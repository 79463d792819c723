"""Small Form A smooths for compute-sanitizer: the dataflow launch (tile_flow) and the per-pass
kernels (stream driver), checked against the oracle.  Usage:
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_flow.py"""
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
