mkdir -p gpurun_out
export TSG_SEGV_TRACE=1
timeout 1800 python -m pytest tests/test_gpu_topology.py tests/test_gpu_api.py tests/test_gpu_quality.py -x -q --durations=5 > gpurun_out/pytest_c16.log 2>&1; echo pytest_rc=$?; tail -12 gpurun_out/pytest_c16.log
python - <<'PY'
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1502_00355_b200 as ts
from paper_1502_00355_b200 import capi
xy, tri = ts.graded_arrays(16_000_000, 1, 1e-3, 1024)
ctx = capi.Context(0)
for rep in range(2):
    t = time.time(); d = ctx.topology(len(xy), tri); td = time.time() - t
    t = time.time(); h = ts.topology(len(xy), tri); th = time.time() - t
    print(f"cfg3 topology: device {td:.2f} s, host {th:.2f} s", flush=True)
t = time.time(); order = capi.hilbert_order(xy); print(f"hilbert {time.time()-t:.2f} s")
t = time.time(); dm = capi.DeviceMesh(ctx, xy, tri, d, order=order); print(f"upload (host layout prep + H2D) {time.time()-t:.2f} s")
PY
