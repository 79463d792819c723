"""GPU parity at the BASELINE.json sizes, through the C ABI (libtsg.so).

The small-mesh suite (test_gpu_parity.py) pins every code path bit for bit; this file checks
the same contract on the meshes the benchmark numbers are quoted on, where the scale-only
hazards live: tile staging caps, u32 word offsets, hub counts, the AUTO side-row schedule
(at 16M nodes rows of valence 257..1024 run in the persistent side kernel's chunked branch,
which smaller meshes route to hub CTAs), graph reuse over millions of tiles.

References, all the reference's own outputs:
  * cfg2 (1M Delaunay, seed 42): the committed digests tests/golden/golden_big.json
    (d1m_formA_10: made by the reference build, tests/golden/make_golden.py);
  * cfg2 Form B W=148, cfg3 (16M graded) and cfg4 (64M grid): the reference's own smooth()
    (oracle/_ref/libtsref.so, compiled from proj/src) run in the test on the same mesh, with
    Backend::Parallel over all host cores (bitwise equal to serial for Form A,
    proj/tests/acceptance.cpp:146-193; W-chunk semantics for Form B).
fp64 parity is bit-exact: coordinates, accepted_per_pass, max_disp_per_pass (hex), triangle α
field and vertex minima (proj/src/smoothing.cpp:76-142, :146-182).
"""
import numpy as np
import pytest

from helpers import sha

pytestmark = pytest.mark.gpu


def _device_run(capi, ctx, ts, xy, tri, topo, form="a", strategy="fused", chunks=1, passes=3, layout="aos",
                swap="pingpong", reorder=True, driver="graph", side=None, precision="f64"):
    order = capi.hilbert_order(xy) if reorder else None
    dm = capi.DeviceMesh(ctx, xy, tri, topo, layout=layout, precision=precision, order=order)
    if side:
        dm.side_schedule(side)
    cfg = capi.make_cfg(form=form, strategy=strategy, chunks=chunks, swap=swap, max_iters=passes, driver=driver,
                        move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy))
    res = dm.smooth(cfg)
    res["xy"] = dm.get_coords()
    return dm, res


def _assert_same(res, want, what):
    assert res["iterations"] == want.iterations, what
    assert np.array_equal(res["accepted"], want.accepted), (what, res["accepted"], want.accepted)
    assert np.array_equal(res["max_disp"].view(np.uint64), want.max_disp.view(np.uint64)), what
    bad = np.flatnonzero((res["xy"].view(np.uint64) != want.xy.view(np.uint64)).any(axis=1))
    assert bad.size == 0, f"{what}: {bad.size} vertices differ, first {bad[:8]}"


@pytest.fixture(scope="module")
def d1m(ts):
    xy, tri = ts.delaunay_arrays(1_000_000, 42)
    return xy, tri, ts.topology(len(xy), tri)


@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_cfg2_1m_fp32(capi, gpu_ctx, ts, port, golden_big, d1m, layout):
    """cfg2 in fp32 (the staged tile path with 8-byte coordinate pairs): one pass in lockstep
    with the oracle's f64 pass (decisions equal except where the f64 margin is within 1e-4),
    and a 10-pass graph smooth whose acceptance counts track the reference's fp64 ones."""
    xy, tri, topo = d1m
    state = np.array(xy, dtype=np.float32).astype(np.float64)
    dm = capi.DeviceMesh(gpu_ctx, state, tri, topo, layout=layout, precision="f32",
                         order=capi.hilbert_order(xy))
    dec, acc, _ = dm.pass_lockstep(form="a")
    _, wdec, margin = port.pass_lockstep(topo, tri, state, form="a", chunks=1, precision=0)
    assert np.array_equal(dec < 0, wdec < 0)
    differ = (wdec >= 0) & (dec != wdec)
    assert not (differ & (margin > 1e-4)).any()
    assert acc == int((dec == 1).sum())
    dm.set_coords(state)
    res = dm.smooth(capi.make_cfg(form="a", max_iters=10, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy)))
    # fp32 resolves moves down to ~1e-7 of the coordinates: from pass ~8 on, moves the fp64
    # run still accepts are ties in fp32 and the counts drift apart (measured: -13% at pass
    # 10), so only the first six passes are held to 1%.
    want = np.array(golden_big["d1m_formA_10"]["accepted"], dtype=np.float64)
    assert res["iterations"] == 10
    got = np.asarray(res["accepted"], dtype=np.float64)
    assert np.all(np.abs(got[:6] - want[:6]) <= 1e-2 * want[:6])
    assert np.all(got <= want * 1.01)
    dm.free()


@pytest.mark.parametrize("variant", [
    dict(layout="aos", reorder=True),                       # the bench configuration
    dict(layout="soa", reorder=True),
    dict(layout="aos", reorder=False, swap="copy"),
    dict(layout="soa", reorder=True, strategy="twophase"),
    dict(layout="aos", reorder=True, driver="stream"),
])
def test_cfg2_1m_form_a_matches_reference_golden(capi, gpu_ctx, ts, golden_big, d1m, variant):
    """cfg2: 1M random Delaunay (seed 42), 10 Form A passes == the reference's digests."""
    case = golden_big["d1m_formA_10"]
    xy, tri, topo = d1m
    assert sha(xy) == case["xy_in"] and sha(tri) == case["tri"]
    dm, res = _device_run(capi, gpu_ctx, ts, xy, tri, topo, passes=10, **variant)
    assert res["iterations"] == 10 and res["stop"] == "max_iters"
    assert [int(a) for a in res["accepted"]] == case["accepted"]
    assert [float(x).hex() for x in res["max_disp"]] == case["max_disp"]
    assert sha(res["xy"]) == case["xy_out"]
    assert sha(dm.tri_alpha()) == case["tri_alpha"]
    assert sha(dm.vertex_minima()) == case["vertex_min"]
    dm.free()


@pytest.mark.parametrize("layout,strategy", [("aos", "fused"), ("soa", "twophase")])
def test_cfg2_1m_form_b_w148_matches_reference(capi, gpu_ctx, ts, ref, d1m, layout, strategy):
    """cfg2 in Form B with W = 148 chunks (one per SM): the reference's Backend::Parallel with
    148 workers (proj/include/trismooth/parallel.hpp:19-24 chunking), 4 passes."""
    xy, tri, topo = d1m
    want = ref.smooth(xy, tri, form="b", strategy=strategy, backend="parallel", workers=148, max_iters=4,
                      move_tol=0.0, layout=layout)
    dm, res = _device_run(capi, gpu_ctx, ts, xy, tri, topo, form="b", strategy=strategy, chunks=148, passes=4,
                          layout=layout, reorder=False)
    _assert_same(res, want, f"cfg2 form B W=148 {layout} {strategy}")
    dm.free()


def _ref_workers(ref):
    return max(1, ref.hardware_concurrency())


def test_cfg3_16m_graded_matches_reference(capi, gpu_ctx, ts, ref):
    """cfg3, the headline mesh: 16M-node graded Delaunay (0.1 % hubs, valence up to 1024), the
    bench configuration (Hilbert slots, AoS, fused, ping-pong, graph driver, AUTO side-row
    schedule), 3 passes, bitwise against the reference's smooth() on the same mesh — and the
    per-tier schedule (hub CTAs) on the same device mesh."""
    xy, tri = ts.graded_arrays(16_000_000, 1, 1e-3, 1024)
    topo = ts.topology(len(xy), tri)
    deg = np.diff(topo["nbr_off"])
    assert deg.max() == 1024 and int((deg > 256).sum()) > 0
    w = _ref_workers(ref)
    want = ref.smooth(xy, tri, form="a", strategy="fused", backend="parallel" if w > 1 else "serial", workers=w,
                      max_iters=3, move_tol=0.0, layout="aos")
    dm, res = _device_run(capi, gpu_ctx, ts, xy, tri, topo, passes=3)
    _assert_same(res, want, "cfg3 graph AUTO")
    assert sha(dm.tri_alpha()) == sha(want.tri_alpha)
    vmin = dm.vertex_minima()
    assert np.array_equal(vmin.view(np.uint64), want.vertex_min.view(np.uint64))
    for side, driver in (("kernels", "graph"), ("persist", "stream")):
        dm.set_coords(xy)
        dm.side_schedule(side)
        r = dm.smooth(capi.make_cfg(form="a", max_iters=3, move_tol=0.0, driver=driver))
        r["xy"] = dm.get_coords()
        _assert_same(r, want, f"cfg3 side={side} driver={driver}")
    dm.free()


def test_cfg4_64m_grid_matches_reference(capi, gpu_ctx, ts, ref):
    """cfg4: 64M-node perturbed grid (8000 x 8000), fp64 Form A, 2 passes, bitwise against the
    reference's smooth() (the largest mesh the reference can hold: ~20 GB host RAM)."""
    xy, tri = ts.grid_arrays(8000, 8000, 0.3, 1)
    w = _ref_workers(ref)
    want = ref.smooth(xy, tri, form="a", strategy="fused", backend="parallel" if w > 1 else "serial", workers=w,
                      max_iters=2, move_tol=0.0, layout="aos")
    topo = ts.topology(len(xy), tri)
    dm, res = _device_run(capi, gpu_ctx, ts, xy, tri, topo, passes=2)
    del topo
    _assert_same(res, want, "cfg4")
    dm.free()


def test_dataflow_launch_at_3m_vs_oracle(capi, gpu_ctx, ts, port):
    """A 3M-node mesh takes the Form A dataflow launch under AUTO (at most 12 waves of
    1280-slot tiles, no side rows): bit-identical to the oracle over 6 passes, with the
    no-moves / max-iters bookkeeping of the device stop rule."""
    xy, tri = ts.delaunay_arrays(3_000_000, 17)
    dm = capi.DeviceMesh(gpu_ctx, xy, tri, None, order=capi.hilbert_order(xy))
    res = dm.smooth(capi.make_cfg(form="a", max_iters=6, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy)))
    assert res["schedule"] == "flow"
    want = port.smooth(xy, tri, form="a", max_iters=6, move_tol=0.0)
    assert [int(a) for a in res["accepted"]] == [int(a) for a in want.accepted]
    assert np.array_equal(res["max_disp"].view(np.uint64), want.max_disp.view(np.uint64))
    assert np.array_equal(dm.get_coords().view(np.uint64), want.xy.view(np.uint64))
    dm.free()
