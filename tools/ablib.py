"""Interleaved A/B of libtsg builds on one mesh (less box-to-box noise than separate bench runs).
usage: python tools/ablib.py [--config cfg3] [--reps 4] [--steps 5] lib1.so[:side] lib2.so[:side] ...
(side = auto | kernels | persist: the mesh's side-row schedule)
Each library gets its own context + device mesh; rounds alternate between them; prints the
per-pass time (device events around each 100-pass smooth) per library: median and min."""
import argparse
import ctypes as C
import statistics
import sys

sys.path.insert(0, ".")
import bench
import paper_1502_00355_b200 as ts
from paper_1502_00355_b200 import capi

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("libs", nargs="+")
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
xy, tri, _ = bench.make_mesh(ts, cfg, None)
topo = ts.topology(len(xy), tri)
order = capi.hilbert_order(xy)
runs = []
for spec in args.libs:
    path, _, side = spec.partition(":")
    capi._lib = None
    capi.LIB_PATH = path
    L = capi.lib()
    ctx = capi.Context(0)
    dm = capi.DeviceMesh(ctx, xy, tri, topo, order=order, precision=cfg["precision"], layout=cfg["layout"])
    scfg = capi.make_cfg(form=cfg["form"], strategy=cfg["strategy"], max_iters=cfg["passes"], move_tol=0.0,
                         bbox_diag=ts.bbox_diagonal(xy))
    if side:
        dm.side_schedule(side)
    runs.append((spec, L, ctx, dm, scfg, []))
for rep in range(args.reps + 1):
    for path, L, ctx, dm, scfg, res in runs:
        capi._lib = L
        for _ in range(args.steps):
            dm.restore_coords()
            r = dm.smooth(scfg)
            if rep > 0:  # round 0 = warm-up
                res.append(r["device_ms"] / r["iterations"])
for path, L, ctx, dm, scfg, res in runs:
    print(f"{path.split('/')[-1]:32s} ms/pass median {statistics.median(res):.4f} min {min(res):.4f} "
          f"max {max(res):.4f} (n={len(res)})")
