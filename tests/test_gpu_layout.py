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


@pytest.mark.parametrize("tile", [768, 1024, 1280])
def test_tile_sizes(capi, gpu_ctx, ts, golden, monkeypatch, tile):
    """Slots per tile are chosen per mesh among the compiled sizes (tsg_engine.cu choose_tile);
    TSG_TILE forces one.  Every size gives the same layout on both preps and the reference's
    exact smoothing (golden d100k_formA_20, reordered and not, AoS and SoA)."""
    from helpers import fixture, sha, smooth_kwargs_to_capi

    monkeypatch.setenv("TSG_TILE", str(tile))
    for name, (xy, tri) in list(_cases(ts))[:3]:
        topo = ts.topology(len(xy), tri)
        assert gpu_ctx.layout_check(xy, tri, topo, capi.hilbert_order(xy)) == "", name
    case = golden["cases"]["d100k_formA_20"]
    xy, tri = fixture(ts, case["kind"], case["args"])
    kw = smooth_kwargs_to_capi(case["smooth"])
    topo = ts.topology(len(xy), tri)
    for order in (capi.hilbert_order(xy), None):
        for precision_layout in ("aos", "soa"):
            dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo, layout=precision_layout, order=order)
            cfg = capi.make_cfg(form=kw["form"], strategy=kw["strategy"], max_iters=kw["max_iters"],
                                move_tol=kw["move_tol"], bbox_diag=ts.bbox_diagonal(xy))
            res = dm.smooth(cfg)
            assert [int(a) for a in res["accepted"]] == case["accepted"]
            assert sha(dm.get_coords()) == case["xy_out"]
            dm.free()


def test_unsupported_tile_size_is_rejected(capi, gpu_ctx, ts, monkeypatch):
    monkeypatch.setenv("TSG_TILE", "1000")
    xy, tri = ts.delaunay_arrays(2000, 1)
    with pytest.raises(RuntimeError, match="TSG_TILE"):
        capi.DeviceMesh(gpu_ctx, xy, tri, ts.topology(len(xy), tri))


@pytest.mark.parametrize("with_order", [True, False])
def test_upload_from_triangles_equals_upload(capi, gpu_ctx, ts, with_order):
    """tsg_mesh_upload_triangles (adjacency built and consumed on the device) gives the same mesh
    as tsg_mesh_upload with tsg_topology's host arrays: identical smoothing, α field and minima."""
    for name, (xy, tri) in _cases(ts):
        if len(xy) < 16:
            continue
        order = capi.hilbert_order(xy) if with_order else None
        res = []
        for topo in (gpu_ctx.topology(len(xy), tri), None):
            dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo, order=order)
            r = dm.smooth(capi.make_cfg(form="a", max_iters=6, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy)))
            res.append((list(r["accepted"]), dm.get_coords().copy(), dm.tri_alpha().copy(), dm.vertex_minima().copy()))
            dm.free()
        assert res[0][0] == res[1][0], name
        for k in (1, 2, 3):
            assert np.array_equal(res[0][k].view(np.uint64), res[1][k].view(np.uint64)), (name, k)


def test_upload_from_triangles_rejects_bad_corners(capi, gpu_ctx, ts):
    xy, tri = ts.delaunay_arrays(2000, 1)
    bad = tri.copy()
    bad[7, 1] = len(xy)
    with pytest.raises(RuntimeError, match="corner index out of range"):
        capi.DeviceMesh(gpu_ctx, xy, bad, None)
