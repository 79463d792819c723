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
