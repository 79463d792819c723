"""Timeline of one Form A pass on cfg3 from a TSG_TRACE build (make -B tsg EXTRA_NVFLAGS=-DTSG_TRACE).

Prints, per kernel (tile / hub CTA / warp row), the start and end spread relative to the first
tile CTA, and the occupancy of each over time in 20 us bins."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np

import bench
import paper_1502_00355_b200 as ts
from paper_1502_00355_b200 import capi

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"])
xy, tri, _ = bench.make_mesh(ts, cfg, None)
topo = ts.topology(len(xy), tri)
ctx = capi.Context(0)
dm = capi.DeviceMesh(ctx, xy, tri, topo, order=capi.hilbert_order(xy))
scfg = capi.make_cfg(form="a", max_iters=25, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy))
dm.smooth(scfg)
KMAX = 65536
buf = np.zeros((3, KMAX, 2), dtype=np.uint64)
L = capi.lib()
L.tsg_debug_trace.argtypes = [C.c_void_p, C.c_int64]
assert L.tsg_debug_trace(buf.ctypes.data, buf.nbytes) == 0, "not a TSG_TRACE build"
names = ["tile", "hub", "warp"]
t0 = min(int(buf[0][buf[0][:, 0] > 0][:, 0].min()), *(int(b[b[:, 0] > 0][:, 0].min()) for b in buf[1:] if (b[:, 0] > 0).any()))
recs = {}
for k, nm in enumerate(names):
    b = buf[k]
    m = b[:, 0] > 0
    st = (b[m, 0].astype(np.int64) - t0) / 1000.0
    du = (b[m, 1] >> 8).astype(np.int64) / 1000.0
    sm = (b[m, 1] & 0xFF).astype(np.int64)
    recs[nm] = (st, du, sm)
    if len(st):
        print(f"{nm:5s} n={len(st):6d} start [{st.min():7.1f}, {st.max():7.1f}] us  end max {np.max(st + du):7.1f}"
              f"  dur mean {du.mean():6.2f} p50 {np.median(du):6.2f} p99 {np.percentile(du, 99):6.2f} max {du.max():6.2f}")
end = max(np.max(s + d) for s, d, _ in recs.values() if len(s))
bins = np.arange(0, end + 20, 20)
print("\nt(us)   " + "  ".join(f"{n:>6s}" for n in names) + "   (mean resident CTAs/warps)")
for lo in bins[:-1]:
    hi = lo + 20
    row = []
    for nm in names:
        s, d, _ = recs[nm]
        ov = np.clip(np.minimum(s + d, hi) - np.maximum(s, lo), 0, None).sum() / 20.0
        row.append(f"{ov:6.1f}")
    print(f"{lo:6.0f}  " + "  ".join(row))
