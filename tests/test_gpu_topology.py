"""Mesh topology on the device (csrc/tsg_topo.cu, tsg_topology) against the host build pinned to
the reference (paper_1502_00355_b200.topology == find_neighbors / determine_constraints,
proj/src/topology.cpp:12-95, tests/test_host_api.py): identical unique-neighbour rows,
incident rows and boundary flags, bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEYS = ("nbr_off", "nbr", "inc_off", "inc", "boundary")


def _same(a, b):
    for k in KEYS:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


@pytest.mark.parametrize("case", ["grid", "delaunay", "graded", "flipped", "nonmanifold"])
def test_device_topology_equals_host(capi, gpu_ctx, ts, port, case):
    if case == "grid":
        xy, tri = ts.grid_arrays(37, 53, 0.3, 2)
    elif case == "delaunay":
        xy, tri = ts.delaunay_arrays(50000, 3)
    elif case == "graded":
        xy, tri = ts.graded_arrays(60000, 3, 2e-3, 2048)
    elif case == "flipped":
        xy, tri = ts.delaunay_arrays(8000, 5)
        tri = tri.copy()
        f = np.random.default_rng(0).random(len(tri)) < 0.1
        tri[f] = tri[f][:, [0, 2, 1]]
    else:
        # vertex 3 isolated; edge (0, 1) shared by three triangles
        xy = np.array([[0, 0], [1, 0], [0, 1], [5, 5], [0.5, -1], [0.5, 1.5]], dtype=np.float64)
        tri = np.array([[0, 1, 2], [1, 0, 4], [0, 1, 5]], dtype=np.int32)
    got = gpu_ctx.topology(len(xy), tri)
    _same(got, ts.topology(len(xy), tri))
    _same(got, port.topology(len(xy), tri))


def test_device_topology_at_cfg3_scale(gpu_ctx, ts):
    """The 16M-node graded mesh of the headline config (valence up to 1024)."""
    xy, tri = ts.graded_arrays(16_000_000, 1, 1e-3, 1024)
    _same(gpu_ctx.topology(len(xy), tri), ts.topology(len(xy), tri))


def test_device_topology_rejects_bad_corners(gpu_ctx):
    with pytest.raises(RuntimeError, match="corner index out of range"):
        gpu_ctx.topology(3, np.array([[0, 1, 3]], dtype=np.int32))
