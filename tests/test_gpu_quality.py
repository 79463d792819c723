"""Quality audit on the device (csrc/tsg_quality.cu) against the reference's definitions.

References:
  * triangle_alpha (proj/include/trismooth/quality.hpp:15-23) restated in numpy below —
    elementwise IEEE float64 in the reference's operand order with no FMA contraction, so it
    is bit-exact — and pinned to the reference's own triangle_alpha on a sample
    (oracle/_ref via the `ref` fixture);
  * the folds of quality_summary / `trismooth quality` (proj/bindings/module.cpp:157-185,
    proj/tools/main.cpp:151-208) and reduce_vertex_minima (quality.hpp:78-89) restated as
    plain Python loops on small cases, vectorised equivalents on large ones.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

K = 2.0 * 1.7320508075688772935


def alpha_np(xy, tri):
    p1, p2, p3 = xy[tri[:, 0]], xy[tri[:, 1]], xy[tri[:, 2]]
    ax, ay = p2[:, 0] - p1[:, 0], p2[:, 1] - p1[:, 1]
    bx, by = p3[:, 0] - p1[:, 0], p3[:, 1] - p1[:, 1]
    cx, cy = p3[:, 0] - p2[:, 0], p3[:, 1] - p2[:, 1]
    ta = ax * by - ay * bx
    es = ((((ax * ax + ay * ay) + bx * bx) + by * by) + cx * cx) + cy * cy
    with np.errstate(invalid="ignore", divide="ignore"):
        q = (K * ta) / es
    return np.where(es == 0.0, 0.0, q)


def fold_report(alpha):
    """The reference's sequential folds, literally (tools/main.cpp:159-172)."""
    lo, hi, nonpos, bins = 2.0, -2.0, 0, [0] * 20
    for q in alpha.tolist():
        lo = q if q < lo else lo
        hi = q if hi < q else hi
        nonpos += q <= 0.0
        b = int((q + 1.0) * 10.0) if q == q else -(2 ** 31)
        bins[min(19, max(0, b))] += 1
    return lo, hi, nonpos, bins


def same_bits(a, b):
    return np.array_equal(np.asarray(a, dtype=np.float64).view(np.uint64), np.asarray(b, dtype=np.float64).view(np.uint64))


def test_alpha_restatement_is_pinned_to_the_reference(ts, ref):
    xy, tri = ts.delaunay_arrays(2000, 3)
    want = np.array([ref.alpha(tuple(xy[a]), tuple(xy[b]), tuple(xy[c])) for a, b, c in tri])
    assert same_bits(alpha_np(xy, tri), want)


@pytest.mark.parametrize("n", [5000, 1_000_000])
def test_tri_alpha_field_and_report(ts, gpu_ctx, n):
    xy, tri = ts.delaunay_arrays(n, 42)
    alpha, rep = gpu_ctx.quality_tri_alpha(xy, tri)
    want = alpha_np(xy, tri)
    assert same_bits(alpha, want)
    assert same_bits(rep["min_alpha"], want.min()) and same_bits(rep["max_alpha"], want.max())
    assert rep["non_positive"] == int((want <= 0).sum())
    bins = np.clip(((want + 1.0) * 10.0).astype(np.int64), 0, 19)
    assert rep["histogram"] == np.bincount(bins, minlength=20).tolist()


@pytest.mark.parametrize("first", ["neg", "pos"])
def test_report_folds_signed_zero_nan_and_degenerate(gpu_ctx, first):
    """Ties keep the FIRST triangle (the sign of a zero extreme), NaN never replaces, a
    zero-size triangle has α = +0 (quality.hpp:21)."""
    xy = np.array([[0, 0], [-1, 0], [2, 0], [1, 0], [0.5, 0.8], [np.nan, 0.0], [3, 3]], dtype=np.float64)
    neg = [0, 1, 2]   # ax*by = -0, ay*bx = +0 -> ta = -0 -> α = -0.0
    pos = [0, 3, 2]   # collinear, ta = +0 -> α = +0.0
    tris = [neg, pos] if first == "neg" else [pos, neg]
    tris = tris + [[6, 6, 6], [0, 3, 4], [5, 0, 3], [0, 1, 4]]
    tri = np.array(tris, dtype=np.int32)
    alpha, rep = gpu_ctx.quality_tri_alpha(xy, tri)
    want = alpha_np(xy, tri)
    assert same_bits(alpha, want)
    lo, hi, nonpos, bins = fold_report(want)
    assert same_bits(rep["min_alpha"], lo) and same_bits(rep["max_alpha"], hi)
    assert rep["non_positive"] == nonpos and rep["histogram"] == bins
    # the inverted triangle (0, 1, 4) makes the minimum; drop it to make zero the minimum
    alpha2, rep2 = gpu_ctx.quality_tri_alpha(xy, tri[:-1])
    lo2, _, _, _ = fold_report(alpha_np(xy, tri[:-1]))
    assert lo2 == 0.0 and math.copysign(1.0, lo2) == (-1.0 if first == "neg" else 1.0)
    assert same_bits(rep2["min_alpha"], lo2)


def test_vertex_minima_fold(ts, gpu_ctx):
    xy, tri = ts.delaunay_arrays(20000, 9)
    xy = np.vstack([xy, [[5.0, 5.0]]])  # isolated vertex -> NaN (kUnsetQuality)
    topo = ts.topology(len(xy), tri)
    alpha = alpha_np(xy, tri)
    alpha[::97] = np.nan  # stored NaN slots never replace a minimum
    got = gpu_ctx.quality_vertex_minima(topo["inc_off"], topo["inc"], alpha)
    want = np.empty(len(xy))
    off, inc = topo["inc_off"], topo["inc"]
    for v in range(len(xy)):
        if off[v] == off[v + 1]:
            want[v] = np.nan
            continue
        lowest = math.inf
        for t in inc[off[v]:off[v + 1]].tolist():
            q = alpha[t]
            lowest = q if q < lowest else lowest
        want[v] = lowest
    assert same_bits(got, want)


def test_quality_summary_matches_reference_definition(ts, port):
    for layout in ("aos", "soa"):
        m = ts.generate_delaunay(3000, seed=2, layout=layout)
        q = ts.quality_summary(m)
        assert set(q) == {"min_alpha", "mean_alpha", "max_alpha", "non_positive", "boundary_vertices",
                          "interior_vertices"}
        xy = np.array(m.points(), dtype=np.float64)
        tri = np.array(m.triangles(), dtype=np.int32)
        want = alpha_np(xy, tri)
        assert same_bits(m.tri_alphas(), want)  # written back into the mesh
        assert same_bits(q["min_alpha"], want.min()) and same_bits(q["max_alpha"], want.max())
        assert same_bits(q["mean_alpha"], np.cumsum(want)[-1] / len(want))  # sequential sum
        bnd = port.topology(len(xy), tri)["boundary"]
        assert q["boundary_vertices"] == int(bnd.sum())
        assert q["interior_vertices"] == len(xy) - int(bnd.sum())
        rep = ts.quality_report(m)
        assert sum(rep["histogram_bins"]) == len(tri) and same_bits(rep["mean_alpha"], q["mean_alpha"])


def test_two_phase_update_after_smooth(ts):
    """update_two_phase on a mesh whose adjacency smooth() installed: the α field and vertex
    minima equal what smooth() wrote back (the reference syncs both to the final coords)."""
    m = ts.generate_delaunay(4000, seed=6)
    ts.smooth(m, form="a", max_iters=5, move_tol=0.0)
    a0, v0 = np.array(m.tri_alphas()), np.array(m.vertex_minima())
    ts.update_two_phase(m)
    assert same_bits(m.tri_alphas(), a0) and same_bits(m.vertex_minima(), v0)
