"""The Python drop-in surface (port of proj/tests/python/test_smoke.py) and host mesh prep.

CPU-only parts run everywhere; the smooth() checks of the reference smoke test need the GPU
and live in tests/test_gpu_api.py.
"""
import math

import numpy as np
import pytest

import trismooth as ts  # the drop-in shim over paper_1502_00355_b200
from helpers import sha


def test_generate_delaunay_counts():
    m = ts.generate_delaunay(300, seed=5)
    assert m.vertex_count == 300
    assert m.triangle_count > 300
    assert m.layout == "aos"
    assert "300 vertices" in repr(m)


def test_generate_is_deterministic():
    a = ts.generate_delaunay(120, seed=9)
    b = ts.generate_delaunay(120, seed=9)
    assert a.points() == b.points()
    assert a.triangles() == b.triangles()
    c = ts.generate_delaunay(120, seed=10)
    assert c.points() != a.points()


def test_triangle_alpha_values():
    assert ts.triangle_alpha((0, 0), (1, 0), (0.5, math.sqrt(3) / 2)) == pytest.approx(1.0)
    assert ts.triangle_alpha((0, 0), (1, 0), (0, 1)) == pytest.approx(math.sqrt(3) / 2)
    assert ts.triangle_alpha((0, 0), (1, 0), (2, 0)) == 0.0
    assert ts.triangle_alpha((0, 0), (0, 1), (1, 0)) == pytest.approx(-math.sqrt(3) / 2)


def test_quality_audit_needs_the_device():
    """quality_summary / compute_all_qualities run on the device audit kernels: without a
    CUDA device they raise (no CPU fallback).  GPU parity: tests/test_gpu_quality.py."""
    import paper_1502_00355_b200 as core

    if core.device_count() > 0:
        pytest.skip("a CUDA device is visible; covered by test_gpu_quality.py")
    m = ts.generate_delaunay(200, seed=2)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        ts.quality_summary(m)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        core.compute_all_qualities(m)


def test_file_round_trip(tmp_path):
    m = ts.generate_delaunay(150, seed=4)
    prefix = str(tmp_path / "mesh")
    ts.write_mesh(m, prefix)
    back = ts.read_mesh(prefix + ".node", prefix + ".ele")
    assert back.points() == m.points()
    assert back.triangles() == m.triangles()


def test_convert_layout():
    m = ts.generate_grid(6, 7, perturbation=0.2, seed=8)
    soa = ts.convert_layout(m, "soa")
    assert soa.layout == "soa"
    assert soa.points() == m.points()
    assert soa.triangles() == m.triangles()
    back = ts.convert_layout(soa, "aos")
    assert back.layout == "aos"
    assert back.points() == m.points()


def test_build_mesh_and_validation():
    m = ts.build_mesh([(0, 0), (1, 0), (0, 1)], [(0, 1, 2)])
    assert m.vertex_count == 3 and m.triangle_count == 1
    with pytest.raises(RuntimeError):
        ts.build_mesh([(0, 0), (1, 0), (0, 1)], [(0, 1, 5)])
    with pytest.raises(RuntimeError):
        ts.build_mesh([(0, 0), (1, 0), (0, 1)], [(0, 1, 1)])
    with pytest.raises(RuntimeError):
        ts.build_mesh([(0, 0), (1, 0), (0, 1)], [])


def test_argument_validation():
    m = ts.generate_delaunay(50, seed=1)
    with pytest.raises(ValueError):
        ts.smooth(m, form="c")
    with pytest.raises(ValueError):
        ts.smooth(m, precision="f16")
    with pytest.raises(ValueError):
        ts.generate_delaunay(50, seed=1, layout="esoteric")
    with pytest.raises(RuntimeError):
        ts.generate_delaunay(2)
    with pytest.raises(RuntimeError):
        ts.generate_grid(1, 5)


def test_read_mesh_missing_file(tmp_path):
    with pytest.raises(RuntimeError):
        ts.read_mesh(str(tmp_path / "no.node"), str(tmp_path / "no.ele"))


def test_read_mesh_one_based_and_comments(tmp_path):
    (tmp_path / "m.node").write_text("# pts\n3 2 1 1\n1 0 0 7 1\n2 1 0 7 1\n3 0 1 7 0 # last\n")
    (tmp_path / "m.ele").write_text("1 3 0\n1 1 2 3\n")
    m = ts.read_mesh(str(tmp_path / "m.node"), str(tmp_path / "m.ele"), layout="soa")
    assert m.points() == [(0.0, 0.0), (1.0, 0.0), (0.0, 1.0)]
    assert m.triangles() == [[0, 1, 2]]
    (tmp_path / "bad.ele").write_text("1 3 0\n0 0 1 9\n")
    with pytest.raises(RuntimeError, match="ele:2"):
        ts.read_mesh(str(tmp_path / "m.node"), str(tmp_path / "bad.ele"))


# ---- generators pinned to the reference (golden digests made from the reference itself) ----

@pytest.mark.parametrize("name", ["grid100_defaults", "d10k_formA_tol0", "d1k_formB_w148", "d300_formA",
                                  "d100k_formA_20", "grid17x23_formA"])
def test_generators_match_reference(golden, name):
    case = golden["cases"][name]
    if case["kind"] == "grid":
        xy, tri = ts.grid_arrays(*case["args"])
    else:
        xy, tri = ts.delaunay_arrays(*case["args"])
    assert sha(xy) == case["xy_in"]
    assert sha(tri) == case["tri"]


def test_delaunay_matches_reference_build(ref):
    for n, seed in ((500, 1), (5000, 2), (30000, 3)):
        xy, tri = ts.delaunay_arrays(n, seed)
        rxy, rtri = ref.delaunay(n, seed)
        assert np.array_equal(xy, rxy) and np.array_equal(tri, rtri)


def test_delaunay_1m_matches_reference(golden_big):
    case = golden_big["d1m_formA_10"]
    xy, tri = ts.delaunay_arrays(1000000, 42)
    assert sha(xy) == case["xy_in"] and sha(tri) == case["tri"]


def test_topology_matches_reference_adjacency(port):
    for xy, tri in (ts.grid_arrays(11, 9, 0.3, 4), ts.delaunay_arrays(3000, 8)):
        a = ts.topology(len(xy), tri)
        b = port.topology(len(xy), tri)
        for k in ("nbr_off", "nbr", "inc_off", "inc", "boundary"):
            assert np.array_equal(a[k], b[k]), k


def test_topology_pins_isolated_and_nonmanifold(port):
    # vertex 3 isolated; edge (0,1) shared by three triangles -> its ends pinned
    xy = np.array([[0, 0], [1, 0], [0, 1], [5, 5], [0.5, -1], [0.5, 1.5]], dtype=np.float64)
    tri = np.array([[0, 1, 2], [1, 0, 4], [0, 1, 5]], dtype=np.int32)
    a = ts.topology(len(xy), tri)
    b = port.topology(len(xy), tri)
    assert np.array_equal(a["boundary"], b["boundary"])
    assert a["boundary"][3] == 1 and a["boundary"][0] == 1 and a["boundary"][1] == 1


def test_graded_generator_heavy_tail():
    xy, tri = ts.graded_arrays(200000, 7, 1e-3, 512)
    topo = ts.topology(len(xy), tri)
    deg = np.diff(topo["nbr_off"])
    interior = topo["boundary"] == 0
    assert len(xy) > 150000
    assert (deg[interior] >= 32).sum() >= 1e-3 * len(xy) * 0.9
    assert deg.max() >= 512
    assert ts.triangulate(xy).shape == tri.shape  # deterministic
    xy2, tri2 = ts.graded_arrays(200000, 7, 1e-3, 512)
    assert np.array_equal(xy, xy2) and np.array_equal(tri, tri2)
    # all CCW, none degenerate
    p = xy[tri]
    area = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - (p[:, 1, 1] - p[:, 0, 1]) * (p[:, 2, 0] - p[:, 0, 0])
    assert (area > 0).all()


def test_bbox_diagonal_matches_reference_formula():
    xy, _ = ts.delaunay_arrays(1000, 3)
    d = ts.bbox_diagonal(xy)
    assert d == math.hypot(xy[:, 0].max() - xy[:, 0].min(), xy[:, 1].max() - xy[:, 1].min())


def _local_delaunay_violations(xy, tri, sample, rng):
    """Edges (of `sample` random triangles) whose opposite vertex across the edge lies strictly
    inside the triangle's circumcircle beyond rounding: local Delaunay on every edge is
    equivalent to the global empty-circumcircle property."""
    nt = len(tri)
    idx = rng.choice(nt, size=min(sample, nt), replace=False)
    # edge -> triangles map via sorted edge keys (all triangles: the neighbour may be anywhere)
    e = np.concatenate([tri[:, [0, 1]], tri[:, [1, 2]], tri[:, [2, 0]]])
    opp = np.concatenate([tri[:, 2], tri[:, 0], tri[:, 1]])
    owner = np.tile(np.arange(nt), 3)
    key = np.minimum(e[:, 0], e[:, 1]).astype(np.int64) * len(xy) + np.maximum(e[:, 0], e[:, 1])
    order = np.argsort(key, kind="stable")
    ks, os_, ow = key[order], opp[order], owner[order]
    pair = np.flatnonzero(ks[1:] == ks[:-1])  # interior edges: two consecutive entries
    sel = np.isin(ow[pair], idx)
    pair = pair[sel]
    a, b = ow[pair], os_[pair + 1]  # triangle a, the vertex opposite across the shared edge
    p = xy[tri[a]]
    d = xy[b]
    ax, ay = p[:, 0, 0] - d[:, 0], p[:, 0, 1] - d[:, 1]
    bx, by = p[:, 1, 0] - d[:, 0], p[:, 1, 1] - d[:, 1]
    cx, cy = p[:, 2, 0] - d[:, 0], p[:, 2, 1] - d[:, 1]
    det = ((ax * ax + ay * ay) * (bx * cy - cx * by) - (bx * bx + by * by) * (ax * cy - cx * ay)
           + (cx * cx + cy * cy) * (ax * by - bx * ay))
    scale = ((ax * ax + ay * ay) * (np.abs(bx * cy) + np.abs(cx * by))
             + (bx * bx + by * by) * (np.abs(ax * cy) + np.abs(cx * ay))
             + (cx * cx + cy * cy) * (np.abs(ax * by) + np.abs(bx * ay)))
    return int((det > 1e-12 * scale).sum()), len(pair)


def test_spatial_insertion_equals_generation_order_at_1m(golden_big):
    """Beyond 2M points the generator inserts along a Hilbert curve; the triangulation must be
    the same canonical output as the reference's generation-order insertion: forced on the 1M
    golden point set it reproduces the reference's triangles exactly."""
    case = golden_big["d1m_formA_10"]
    xy, tri = ts.delaunay_arrays(1_000_000, 42)
    assert sha(tri) == case["tri"]
    spatial = ts.triangulate(xy, True)
    assert sha(spatial) == case["tri"]


def test_spatial_generator_is_delaunay_at_4m():
    """A 4M-point mesh (spatial insertion path): CCW, canonical (smallest corner first, sorted),
    Euler count nt = 2n - 2 - h, and no local Delaunay violation on 200K sampled triangles."""
    xy, tri = ts.delaunay_arrays(4_000_000, 7)
    n = len(xy)
    assert tri.shape[0] > 2 * n - 2 - 4 * int(np.sqrt(n))  # h (hull size) is O(sqrt n)
    assert (tri[:, 0] < tri[:, 1]).all() and (tri[:, 0] < tri[:, 2]).all()
    first = tri[:, 0].astype(np.int64) * n * n + tri[:, 1].astype(np.int64) * n + tri[:, 2]
    assert (np.diff(first) > 0).all()
    p = xy[tri]
    area = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - (p[:, 1, 1] - p[:, 0, 1]) * (p[:, 2, 0] - p[:, 0, 0])
    assert (area > 0).all()
    bad, checked = _local_delaunay_violations(xy, tri, 200_000, np.random.default_rng(1))
    assert checked > 250_000 and bad == 0


def test_binary_mesh_round_trip_and_validation(tmp_path):
    import paper_1502_00355_b200 as core

    xy, tri = ts.delaunay_arrays(20000, 6)
    p = str(tmp_path / "m.tsgmesh")
    core.write_binary(p, xy, tri)
    xy2, tri2 = core.read_binary(p)
    assert np.array_equal(xy.view(np.uint64), xy2.view(np.uint64)) and np.array_equal(tri, tri2)
    raw = bytearray(open(p, "rb").read())
    open(str(tmp_path / "short"), "wb").write(raw[:-4])
    with pytest.raises(RuntimeError, match="do not match"):
        core.read_binary(str(tmp_path / "short"))
    bad = tri.copy()
    bad[5, 1] = len(xy)
    core.write_binary(str(tmp_path / "bad"), xy, bad)
    with pytest.raises(RuntimeError, match="out of range"):
        core.read_binary(str(tmp_path / "bad"))
    open(str(tmp_path / "junk"), "wb").write(b"NOTAMESH" + bytes(40))
    with pytest.raises(RuntimeError, match="not a TSGMESH1"):
        core.read_binary(str(tmp_path / "junk"))
