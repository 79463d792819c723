"""Prep wall times of the two upload paths (host-topology round trip vs tsg_mesh_upload_triangles)
on one mesh, alternating, in one process.  usage: python tools/prep_probe.py [cfg2|cfg3]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1502_00355_b200 as ts  # noqa: E402
from paper_1502_00355_b200 import capi  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
xy, tri = ts.delaunay_arrays(1_000_000, 42) if cfg == "cfg2" else ts.graded_arrays(16_000_000, 1, 1e-3, 1024)
ctx = capi.Context(0)
for rep in range(3):
    for path in ("roundtrip", "fused"):
        t0 = time.time()
        order = ctx.hilbert_order(xy)
        t1 = time.time()
        if path == "roundtrip":
            topo = ctx.topology(len(xy), tri)
            t2 = time.time()
            dm = capi.DeviceMesh(ctx, xy, tri, topo, order=order)
        else:
            t2 = time.time()
            dm = capi.DeviceMesh(ctx, xy, tri, None, order=order)
        t3 = time.time()
        print(f"{cfg} rep {rep} {path:9s} order {t1 - t0:.3f} topology {t2 - t1:.3f} upload {t3 - t2:.3f} total {t3 - t0:.3f}",
              flush=True)
        dm.free()
