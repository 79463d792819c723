"""Device layout prep (csrc/tsg_layout_dev.cu, the default of tsg_mesh_upload) against the host
build (tsg_prep.cpp build_host_mesh, TSG_HOST_PREP=1): every array of the device mesh — slot
order, ranks, compact CSR, fan records, fan16, device triangle order and corners, incident CSR,
tier lists, tile meta / records / externals — identical (tsg_debug_layout_check), so the two
preps give bit-identical smoothing; the parity suites run on the device prep."""
import numpy as np
import pytest

from helpers import fan

pytestmark = pytest.mark.gpu


def _cases(ts):
    xy, tri = ts.delaunay_arrays(6000, 70)
    flip = np.random.default_rng(1).random(len(tri)) < 0.05
    tri_f = tri.copy()
    tri_f[flip] = tri_f[flip][:, [0, 2, 1]]
    yield "grid", ts.grid_arrays(61, 47, 0.3, 2)
    yield "delaunay", ts.delaunay_arrays(40000, 3)
    yield "graded", ts.graded_arrays(60000, 3, 2e-3, 2048)
    yield "flipped", (xy, tri_f)
    yield "fan5000", fan(5000, (0.01, -0.02))
    yield "tiny", (np.array([[0, 0], [1, 0], [0, 1], [1, 1]], float), np.array([[0, 1, 2], [1, 3, 2]], np.int32))


@pytest.mark.parametrize("with_order", [True, False])
def test_device_layout_equals_host(capi, gpu_ctx, ts, with_order):
    for name, (xy, tri) in _cases(ts):
        topo = ts.topology(len(xy), tri)
        order = capi.hilbert_order(xy) if with_order else None
        assert gpu_ctx.layout_check(xy, tri, topo, order) == "", name


def test_device_layout_equals_host_at_cfg3_scale(capi, gpu_ctx, ts):
    xy, tri = ts.graded_arrays(16_000_000, 1, 1e-3, 1024)
    topo = gpu_ctx.topology(len(xy), tri)
    assert gpu_ctx.layout_check(xy, tri, topo, capi.hilbert_order(xy)) == ""


def test_device_hilbert_order_equals_host(capi, gpu_ctx, ts):
    for xy in (ts.delaunay_arrays(100000, 4)[0], ts.grid_arrays(300, 200, 0.3, 1)[0],
               np.vstack([ts.delaunay_arrays(5000, 1)[0], [[np.nan, 0.5]], [[2.0, 2.0]]])):
        assert np.array_equal(gpu_ctx.hilbert_order(xy), capi.hilbert_order(xy))


def test_device_layout_in_many_sort_chunks(ts):
    """The segmented sorts run in chunks of segments (cfg5 scale); a tiny chunk size forces
    hundreds of chunks on a small mesh (child process: TSG_SEG_CHUNK is read once)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, sys.argv[1]); import paper_1502_00355_b200 as ts; "
            "from paper_1502_00355_b200 import capi; ctx = capi.Context(0); "
            "xy, tri = ts.graded_arrays(50000, 4, 3e-3, 600); topo = ctx.topology(len(xy), tri); "
            "print(repr(ctx.layout_check(xy, tri, topo, capi.hilbert_order(xy))))")
    r = subprocess.run([sys.executable, "-c", code, root], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, TSG_SEG_CHUNK="7"))
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.strip().endswith("''"), r.stdout
