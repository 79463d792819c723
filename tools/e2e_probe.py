import os
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_1502_00355_b200 as ts
from paper_1502_00355_b200 import capi
cfg = dict(bench.CONFIGS["cfg3"])
xy, tri, _ = bench.make_mesh(ts, cfg, 4_000_000)
topo = ts.topology(len(xy), tri)
ctx = capi.Context(0)
dm = capi.DeviceMesh(ctx, xy, tri, topo, order=capi.hilbert_order(xy))
scfg = capi.make_cfg(form="a", max_iters=100, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy))
xin = torch.from_numpy(np.ascontiguousarray(xy)).pin_memory(); xout = torch.empty_like(xin).pin_memory()
a, b = xin.numpy(), xout.numpy()
dm.smooth_host_batch([a], scfg, [b])
for rep in range(6):
    t = time.perf_counter(); its, _ = dm.smooth_host_batch([a] * 10, scfg, [b] * 10); dt = time.perf_counter() - t
    t2 = time.perf_counter(); r = dm.smooth(scfg); torch.cuda.synchronize(); dt2 = time.perf_counter() - t2
    print(f"batch10 {dt*100:.1f} ms/item   single smooth {dt2*1000:.1f} ms  device {r['device_ms']:.1f}")

# host buffers from cudaHostAlloc directly (vs torch pin_memory above)
import ctypes as C
import glob
rt = C.CDLL(sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
def pinned(shape):
    p = C.c_void_p()
    assert rt.cudaHostAlloc(C.byref(p), C.c_size_t(int(np.prod(shape)) * 8), 0) == 0
    return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=shape)
a2, b2 = pinned(xy.shape), pinned(xy.shape)
a2[:] = xy
for rep in range(3):
    t = time.perf_counter(); dm.smooth_host_batch([a2] * 10, scfg, [b2] * 10); dt = time.perf_counter() - t
    print(f"cudaHostAlloc buffers: batch10 {dt*100:.1f} ms/item")
pa, pb = np.ascontiguousarray(xy), np.empty_like(xy)
t = time.perf_counter(); dm.smooth_host_batch([pa] * 10, scfg, [pb] * 10); dt = time.perf_counter() - t
print(f"pageable buffers: batch10 {dt*100:.1f} ms/item")
t = time.perf_counter()
for _ in range(10):
    dm.smooth_host(a, scfg, b)
dt = time.perf_counter() - t
print(f"smooth_host x10 (serial copies): {dt*100:.1f} ms/item")
