"""The bench's e2e leg on cfg3 (tsg_smooth_host_batch, 2 items of 3 passes) for an ncu launch
list of the reorder kernels.  usage: ncu ... python tools/e2e_probe.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1502_00355_b200 as ts  # noqa: E402
from paper_1502_00355_b200 import capi  # noqa: E402

xy, tri = ts.graded_arrays(16_000_000, 1, 1e-3, 1024)
ctx = capi.Context(0)
dm = capi.DeviceMesh(ctx, xy, tri, None, order=ctx.hilbert_order(xy))
xin = torch.from_numpy(np.ascontiguousarray(xy)).pin_memory().numpy()
xout = torch.empty(xy.shape, dtype=torch.float64).pin_memory().numpy()
cfg = capi.make_cfg(form="a", max_iters=3, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy))
dm.smooth_host_batch([xin, xin], cfg, [xout, xout])
print("e2e probe done")
