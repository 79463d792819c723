"""Repeatability of the batch host-buffer path (the bench's e2e leg) on cfg3: per-call ms/item."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_1502_00355_b200 as ts
from paper_1502_00355_b200 import capi
cfg = dict(bench.CONFIGS["cfg3"])
n = int(sys.argv[1]) if len(sys.argv) > 1 else None
xy, tri, _ = bench.make_mesh(ts, cfg, n)
topo = ts.topology(len(xy), tri)
ctx = capi.Context(0)
dm = capi.DeviceMesh(ctx, xy, tri, topo, order=capi.hilbert_order(xy))
scfg = capi.make_cfg(form="a", max_iters=100, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy))
xin = torch.from_numpy(np.ascontiguousarray(xy)).pin_memory(); xout = torch.empty_like(xin).pin_memory()
a, b = xin.numpy(), xout.numpy()
dm.smooth_host_batch([a], scfg, [b])
for rep in range(8):
    t = time.perf_counter(); its, _ = dm.smooth_host_batch([a] * 5, scfg, [b] * 5); dt = time.perf_counter() - t
    t2 = time.perf_counter(); r = dm.smooth(scfg); torch.cuda.synchronize(); dt2 = time.perf_counter() - t2
    print(f"batch5 {dt*200:.1f} ms/item its={list(its)}  single smooth {dt2*1000:.1f} ms  device {r['device_ms']:.1f}", flush=True)
