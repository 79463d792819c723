"""GPU parity tests: the sm_100a path through the C ABI (libtsg.so) against the reference.

fp64 parity is BIT-EXACT (coordinates, accepted_per_pass, max_disp_per_pass, iterations,
stop reason, triangle alpha field, vertex minima): SURVEY §8c.  References:
  * committed golden digests produced by the reference itself (tests/golden/make_golden.py);
  * the oracle restatement (oracle/liboracle.so, itself pinned to the reference in
    tests/test_oracle.py) on fresh seeded meshes.
fp32 parity is lockstep: from the same state, decisions agree except where the
f64 margin |hyp - thr| <= EPS_F32, and positions agree to 1e-5 relative.
"""
import numpy as np
import pytest

from helpers import fan, fixture, sha, smooth_kwargs_to_capi

pytestmark = pytest.mark.gpu

EPS_F32 = 1e-4          # decision margin below which an fp32 flip is allowed
REL_F32 = 1e-5          # coordinate tolerance, relative to the bbox diagonal, fp32 lockstep

GOLDEN_CASES = ["grid100_defaults", "grid100_formA_tol0", "d10k_formA_tol0", "d10k_formB_w8_soa_tol0",
                "d10k_formB_serial_conv", "d10k_formA_serial_conv", "d10k_formB_w3_fused", "d1k_formB_w148",
                "grid17x23_formA", "grid12_formB_loose", "d300_formA", "d100k_formA_20"]


def run_capi(capi, ctx, ts, xy, tri, form, strategy="fused", chunks=1, max_iters=100, move_tol=0.0,
             layout="aos", swap="pingpong", driver="graph", reorder=False, precision="f64"):
    topo = ts.topology(len(xy), tri)
    order = capi.hilbert_order(xy) if reorder else None
    dm = capi.DeviceMesh(ctx, xy, tri, topo, layout=layout, precision=precision, order=order)
    cfg = capi.make_cfg(form=form, strategy=strategy, chunks=chunks, swap=swap, max_iters=max_iters,
                        driver=driver, move_tol=move_tol, bbox_diag=ts.bbox_diagonal(xy))
    res = dm.smooth(cfg)
    res["xy"] = dm.get_coords()
    return dm, res


def assert_case(res, case):
    assert res["iterations"] == case["iterations"]
    assert res["stop"] == case["stop"]
    assert [int(a) for a in res["accepted"]] == case["accepted"]
    assert [float(x).hex() for x in res["max_disp"]] == case["max_disp"]
    assert sha(res["xy"]) == case["xy_out"]


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_golden_case_default_variant(capi, gpu_ctx, ts, golden, name):
    case = golden["cases"][name]
    xy, tri = fixture(ts, case["kind"], case["args"])
    kw = smooth_kwargs_to_capi(case["smooth"])
    dm, res = run_capi(capi, gpu_ctx, ts, xy, tri, kw["form"], kw["strategy"], kw["chunks"], kw["max_iters"],
                       kw["move_tol"], kw["layout"])
    assert_case(res, case)
    assert sha(dm.tri_alpha()) == case["tri_alpha"]
    assert sha(dm.vertex_minima()) == case["vertex_min"]
    dm.free()


VARIANTS = [
    dict(layout="soa"), dict(layout="aos", strategy="twophase"), dict(layout="soa", strategy="twophase"),
    dict(swap="copy"), dict(driver="stream"), dict(layout="soa", swap="copy", driver="stream", strategy="twophase"),
]


@pytest.mark.parametrize("name", ["grid100_formA_tol0", "d10k_formB_w8_soa_tol0", "d10k_formB_serial_conv",
                                  "d10k_formA_serial_conv", "grid12_formB_loose", "d1k_formB_w148"])
@pytest.mark.parametrize("variant", range(len(VARIANTS)))
def test_golden_case_all_variants(capi, gpu_ctx, ts, golden, name, variant):
    """Layouts, strategies, swap forms and drivers change the schedule, never the result."""
    case = golden["cases"][name]
    xy, tri = fixture(ts, case["kind"], case["args"])
    kw = smooth_kwargs_to_capi(case["smooth"])
    v = dict(strategy=kw["strategy"], layout=kw["layout"])
    v.update(VARIANTS[variant])
    dm, res = run_capi(capi, gpu_ctx, ts, xy, tri, kw["form"], chunks=kw["chunks"], max_iters=kw["max_iters"],
                       move_tol=kw["move_tol"], **v)
    assert_case(res, case)
    dm.free()


@pytest.mark.parametrize("name", ["grid100_formA_tol0", "d10k_formA_tol0", "d100k_formA_20", "d10k_formA_serial_conv"])
@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_form_a_locality_reorder_is_invisible(capi, gpu_ctx, ts, golden, name, layout):
    """Hilbert relabelling on the device keeps neighbour sums in original-id order (K10)."""
    case = golden["cases"][name]
    xy, tri = fixture(ts, case["kind"], case["args"])
    kw = smooth_kwargs_to_capi(case["smooth"])
    dm, res = run_capi(capi, gpu_ctx, ts, xy, tri, "a", max_iters=kw["max_iters"], move_tol=kw["move_tol"],
                       layout=layout, reorder=True)
    assert_case(res, case)
    assert sha(dm.tri_alpha()) == case["tri_alpha"]
    assert sha(dm.vertex_minima()) == case["vertex_min"]
    dm.free()


@pytest.mark.parametrize("seed", range(6))
def test_random_meshes_vs_oracle(capi, gpu_ctx, ts, port, seed):
    rng = np.random.default_rng(seed)
    if seed % 2:
        xy, tri = ts.delaunay_arrays(int(rng.integers(500, 40000)), 1000 + seed)
    else:
        xy, tri = ts.grid_arrays(int(rng.integers(5, 120)), int(rng.integers(5, 120)), 0.35, seed)
    form = "ab"[seed % 2 == 0]
    chunks = int(rng.choice([1, 2, 5, 31, 148, 1000]))
    tol = float(rng.choice([0.0, 1e-6, 1e-4]))
    want = port.smooth(xy, tri, form=form, chunks=chunks, max_iters=60, move_tol=tol)
    for layout in ("aos", "soa"):
        dm, got = run_capi(capi, gpu_ctx, ts, xy, tri, form, chunks=chunks, max_iters=60, move_tol=tol,
                           layout=layout, reorder=(form == "a" and layout == "soa"))
        assert got["iterations"] == want.iterations and got["stop"] == want.stop
        assert np.array_equal(got["accepted"], want.accepted)
        assert np.array_equal(got["max_disp"].view(np.uint64), want.max_disp.view(np.uint64))
        assert np.array_equal(got["xy"].view(np.uint64), want.xy.view(np.uint64))
        dm.free()


@pytest.mark.parametrize("form,chunks", [("a", 1), ("b", 1), ("b", 16)])
def test_high_valence_hubs_vs_oracle(capi, gpu_ctx, ts, port, form, chunks):
    """Graded mesh with hub fans (valence 32..2048): the CTA-per-vertex path."""
    xy, tri = ts.graded_arrays(60000, 3, 2e-3, 2048)
    topo = ts.topology(len(xy), tri)
    assert np.diff(topo["nbr_off"]).max() >= 2048
    want = port.smooth(xy, tri, form=form, chunks=chunks, max_iters=15, move_tol=0.0)
    for layout, strategy in (("aos", "fused"), ("soa", "twophase")):
        dm, got = run_capi(capi, gpu_ctx, ts, xy, tri, form, strategy=strategy, chunks=chunks, max_iters=15,
                           layout=layout)
        assert np.array_equal(got["accepted"], want.accepted)
        assert np.array_equal(got["xy"].view(np.uint64), want.xy.view(np.uint64))
        dm.free()


@pytest.mark.parametrize("mode", ["kernels", "persist"])
@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_side_row_schedules_vs_oracle(capi, gpu_ctx, ts, port, mode, layout):
    """Form A fused rows of valence >= 32 either as per-tier grids after the tile grid or in the
    persistent side kernel beside it (ticket counter reused across passes and runs): both
    reproduce the reference bit for bit."""
    xy, tri = ts.graded_arrays(60000, 3, 2e-3, 2048)
    topo = ts.topology(len(xy), tri)
    want = port.smooth(xy, tri, form="a", chunks=1, max_iters=15, move_tol=0.0)
    dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo, layout=layout, order=capi.hilbert_order(xy))
    dm.side_schedule(mode)
    for driver in ("graph", "stream", "graph"):
        dm.set_coords(xy)
        got = dm.smooth(capi.make_cfg(form="a", max_iters=15, move_tol=0.0, driver=driver))
        assert np.array_equal(got["accepted"], want.accepted)
        assert np.array_equal(dm.get_coords().view(np.uint64), want.xy.view(np.uint64))
    dm.free()


@pytest.mark.parametrize("n", [40, 5000, 9000])
def test_single_fan_hub_beyond_shared_memory(capi, gpu_ctx, ts, port, n):
    """A valence above the shared-memory staging cap (4096) reads the tail from global memory."""
    xy, tri = fan(n, (0.013, -0.021))
    xy[0] = (0.3, -0.2)
    for form in ("a", "b"):
        want = port.smooth(xy, tri, form=form, chunks=1, max_iters=3, move_tol=0.0)
        dm, got = run_capi(capi, gpu_ctx, ts, xy, tri, form, max_iters=3)
        assert np.array_equal(got["accepted"], want.accepted)
        assert np.array_equal(got["xy"].view(np.uint64), want.xy.view(np.uint64))
        dm.free()


@pytest.mark.parametrize("mode", ["levels", "chunks", "flow"])
@pytest.mark.parametrize("case", [("grid", (30, 40, 0.3, 2), 1), ("delaunay", (12000, 9), 7),
                                  ("delaunay", (12000, 9), 300)])
def test_form_b_schedules_vs_oracle(capi, gpu_ctx, ts, port, mode, case):
    """The Form B schedules (a launch per dependency level / one CTA per chunk walking its
    levels / the (vertex, pass) dataflow kernel) reproduce the reference bit for bit, both
    strategies."""
    kind, args, chunks = case
    xy, tri = ts.grid_arrays(*args) if kind == "grid" else ts.delaunay_arrays(*args)
    want = port.smooth(xy, tri, form="b", chunks=chunks, max_iters=25, move_tol=0.0)
    for strategy, layout in (("fused", "aos"), ("twophase", "soa")):
        topo = ts.topology(len(xy), tri)
        dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo, layout=layout)
        dm.formb_schedule(mode)
        got = dm.smooth(capi.make_cfg(form="b", strategy=strategy, chunks=chunks, max_iters=25, move_tol=0.0))
        assert np.array_equal(got["accepted"], want.accepted)
        assert np.array_equal(dm.get_coords().view(np.uint64), want.xy.view(np.uint64))
        dm.free()


@pytest.mark.parametrize("case", [((30, 40, 0.3, 2), 1e-5, 1), ((30, 40, 0.3, 2), 1e-5, 7),
                                  ((60, 60, 0.3, 3), 1e-5, 1), ((30, 40, 0.3, 2), 1e-6, 1)])
@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_form_b_dataflow_rounds_and_replay_vs_oracle(capi, gpu_ctx, ts, port, case, layout):
    """The dataflow schedule runs rounds of 64 passes while the displacement stop is live and
    replays the round that stops (tsg_smooth, smooth_flow): stops at passes 71..245, in both
    swap modes, equal the reference's (proj/src/smoothing.cpp:132-141) bit for bit."""
    args, tol, chunks = case
    xy, tri = ts.grid_arrays(*args)
    want = port.smooth(xy, tri, form="b", chunks=chunks, max_iters=1000, move_tol=tol)
    assert 64 < want.iterations < 1000 and want.stop == "displacement"
    topo = ts.topology(len(xy), tri)
    dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo, layout=layout)
    dm.formb_schedule("flow")
    for swap in ("pingpong", "copy"):
        dm.set_coords(xy)
        got = dm.smooth(capi.make_cfg(form="b", chunks=chunks, swap=swap, max_iters=1000, move_tol=tol,
                                      bbox_diag=ts.bbox_diagonal(xy)))
        assert got["iterations"] == want.iterations and got["stop"] == want.stop
        assert np.array_equal(got["accepted"], want.accepted)
        assert np.array_equal(got["max_disp"].view(np.uint64), want.max_disp.view(np.uint64))
        assert np.array_equal(dm.get_coords().view(np.uint64), want.xy.view(np.uint64))
    # round boundaries without a live displacement stop: one launch for all passes
    for n in (63, 64, 65, 129):
        dm.set_coords(xy)
        got = dm.smooth(capi.make_cfg(form="b", chunks=chunks, max_iters=n, move_tol=0.0))
        w = port.smooth(xy, tri, form="b", chunks=chunks, max_iters=n, move_tol=0.0)
        assert got["iterations"] == w.iterations and np.array_equal(got["accepted"], w.accepted)
        assert np.array_equal(dm.get_coords().view(np.uint64), w.xy.view(np.uint64))
    dm.free()


@pytest.mark.parametrize("seed", [0, 1])
def test_mixed_orientation_and_bowtie_links_vs_oracle(capi, gpu_ctx, ts, port, seed):
    """Vertices whose link is not one directed cycle (flipped triangles, a bow-tie vertex shared by
    two fans) take the fan-record sweep of the small tier; the rest take the cycle sweep."""
    rng = np.random.default_rng(seed)
    xy, tri = ts.delaunay_arrays(6000, 70 + seed)
    tri = tri.copy()
    flip = rng.random(len(tri)) < 0.05
    tri[flip] = tri[flip][:, [0, 2, 1]]
    # bow-tie: two separate 4-fans glued at one centre vertex (interior: every edge twice)
    c = len(xy)
    ring = [(0.5 + 0.02 * np.cos(t), 2.5 + 0.02 * np.sin(t)) for t in np.linspace(0, 2 * np.pi, 5)[:-1]]
    ring2 = [(0.501 + 0.03 * np.cos(t), 2.5 + 0.03 * np.sin(t)) for t in np.linspace(0.3, 2 * np.pi + 0.3, 5)[:-1]]
    xy = np.vstack([xy, [[0.501, 2.499]], ring, ring2])
    extra = [[c, c + 1 + k, c + 1 + (k + 1) % 4] for k in range(4)] + \
            [[c, c + 5 + k, c + 5 + (k + 1) % 4] for k in range(4)]
    tri = np.vstack([tri, np.array(extra, np.int32)]).astype(np.int32)
    want = port.smooth(xy, tri, form="a", max_iters=25, move_tol=0.0)
    assert want.accepted[0] > 0
    for layout, reorder in (("aos", True), ("soa", False)):
        dm, got = run_capi(capi, gpu_ctx, ts, xy, tri, "a", max_iters=25, layout=layout, reorder=reorder)
        assert np.array_equal(got["accepted"], want.accepted)
        assert np.array_equal(got["max_disp"].view(np.uint64), want.max_disp.view(np.uint64))
        assert np.array_equal(got["xy"].view(np.uint64), want.xy.view(np.uint64))
        dm.free()


def test_edge_cases(capi, gpu_ctx, ts, port):
    # all-boundary meshes: one pass, no moves (proj/tests/test_smoothing.cpp:142-152)
    for xy, tri in ((np.array([[0, 0], [1, 0], [0, 1]], float), np.array([[0, 1, 2]], np.int32)),
                    (np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float), np.array([[0, 1, 2], [0, 2, 3]], np.int32))):
        dm, r = run_capi(capi, gpu_ctx, ts, xy, tri, "b", max_iters=50, move_tol=1e-6)
        assert r["iterations"] == 1 and r["stop"] == "no_moves" and list(r["accepted"]) == [0]
        assert np.array_equal(r["xy"], xy)
        dm.free()
    # optimal fan is a fixed point: strict acceptance rejects ties (:154-162)
    xy, tri = fan(6, (0.0, 0.0))
    dm, r = run_capi(capi, gpu_ctx, ts, xy, tri, "a", max_iters=10, move_tol=1e-6, layout="soa")
    assert r["stop"] == "no_moves" and r["iterations"] == 1
    assert np.array_equal(r["xy"].view(np.uint64), xy.view(np.uint64))
    dm.free()
    # isolated vertex is pinned, NaN minimum; max_iters = 1 runs one pass
    xy, tri = ts.grid_arrays(6, 6, 0.3, 5)
    xy = np.vstack([xy, [[9.0, 9.0]]])
    dm, r = run_capi(capi, gpu_ctx, ts, xy, tri, "b", max_iters=1)
    want = port.smooth(xy, tri, form="b", max_iters=1, move_tol=0.0)
    assert r["iterations"] == 1 and r["stop"] == "max_iters"
    assert np.array_equal(r["xy"].view(np.uint64), want.xy.view(np.uint64))
    vmin = dm.vertex_minima()
    assert np.isnan(vmin[-1]) and np.array_equal(vmin[:-1], want.vertex_min[:-1])
    dm.free()


def test_repeated_runs_and_graph_reuse_are_deterministic(capi, gpu_ctx, ts):
    xy, tri = ts.delaunay_arrays(20000, 11)
    topo = ts.topology(len(xy), tri)
    dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo)
    cfg = capi.make_cfg(form="b", chunks=7, max_iters=40, move_tol=1e-6, bbox_diag=ts.bbox_diagonal(xy))
    outs = []
    for _ in range(3):
        dm.set_coords(xy)
        r = dm.smooth(cfg)
        outs.append((r["iterations"], dm.get_coords()))
    assert all(o[0] == outs[0][0] and np.array_equal(o[1], outs[0][1]) for o in outs)
    dm.free()


def test_continuing_runs_equal_one_long_run(capi, gpu_ctx, ts, port):
    """Re-running smooth() continues from the device state (stop state restarts)."""
    xy, tri = ts.delaunay_arrays(5000, 4)
    topo = ts.topology(len(xy), tri)
    dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo)
    cfg = capi.make_cfg(form="a", max_iters=7, move_tol=0.0)
    for _ in range(3):
        dm.smooth(cfg)
    want = port.smooth(xy, tri, form="a", max_iters=21, move_tol=0.0)
    assert np.array_equal(dm.get_coords().view(np.uint64), want.xy.view(np.uint64))
    dm.free()


@pytest.mark.parametrize("form,chunks,seed,ordered,layout", [
    ("a", 1, 21, False, "aos"), ("b", 1, 21, False, "aos"), ("b", 64, 21, False, "aos"),
    # Hilbert-ordered meshes run the staged tile path; the seeds give odd and even maximum
    # external counts per tile (fp32 pairs are 8 bytes: the staged words must stay aligned).
    ("a", 1, 21, True, "aos"), ("a", 1, 22, True, "aos"), ("a", 1, 23, True, "aos"), ("a", 1, 24, True, "soa")])
def test_fp32_lockstep(capi, gpu_ctx, ts, port, form, chunks, seed, ordered, layout):
    """fp32: from the oracle's pass-q state, one device pass must make the same decisions except
    where the f64 margin is within EPS_F32, and land within REL_F32 of the f64 positions."""
    xy, tri = ts.delaunay_arrays(30000, seed)
    topo = ts.topology(len(xy), tri)
    diag = ts.bbox_diagonal(xy)
    state = np.array(xy, dtype=np.float32).astype(np.float64)  # f32-representable start
    dm = capi.DeviceMesh(gpu_ctx, state, tri, topo, precision="f32", layout=layout,
                         order=capi.hilbert_order(xy) if ordered else None)
    flips = total = 0
    for q in range(5):
        dm.set_coords(state)
        dec, acc, _ = dm.pass_lockstep(form=form, chunks=chunks)
        got = dm.get_coords()
        want, wdec, margin = port.pass_lockstep(topo, tri, state, form=form, chunks=chunks, precision=0)
        movable = wdec >= 0
        assert np.array_equal(dec < 0, wdec < 0)
        differ = movable & (dec != wdec)
        unexplained = differ & (margin > EPS_F32)
        if form == "a":
            # Jacobi: every input is the shared state, so a flip needs a tiny margin
            assert not unexplained.any(), margin[differ].max()
            same = movable & (dec == wdec)
            err = np.abs(got[same] - want[same]).max() / diag
            assert err <= REL_F32, err
        else:
            # Gauss-Seidel: an upstream flip moves a fresh neighbour, so a few flips cascade
            assert unexplained.sum() <= 1e-3 * movable.sum(), int(unexplained.sum())
        flips += int(differ.sum())
        total += int(movable.sum())
        assert acc == int((dec == 1).sum())
        state = np.array(want, dtype=np.float32).astype(np.float64)
    assert flips <= 0.1 * total
    dm.free()


def test_tri_alpha_and_extrema_device(capi, gpu_ctx, ts, port):
    xy, tri = ts.delaunay_arrays(3000, 5)
    topo = ts.topology(len(xy), tri)
    dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo, layout="soa", order=capi.hilbert_order(xy))
    alpha = dm.tri_alpha()
    want = np.array([port.alpha(tuple(xy[a]), tuple(xy[b]), tuple(xy[c])) for a, b, c in tri])
    assert np.array_equal(alpha.view(np.uint64), want.view(np.uint64))
    lo, hi, nonpos = dm.alpha_extrema()
    assert lo == want.min() and hi == want.max() and nonpos == int((want <= 0).sum())
    dm.free()


def test_fast_alpha_error_is_far_inside_the_guard(gpu_ctx):
    """The decision fast path (SFU reciprocal + 2 Newton steps) must stay far inside its 2^-45
    guard band (8x margin), otherwise a near-tie could be settled wrongly instead of falling back to IEEE
    division.  (One Newton step measures ~2^-40 on this hardware: not enough, hence two.)"""
    err, nonfinite = gpu_ctx.selftest_alpha(1 << 22, 7, 2)
    assert err <= 2.0 ** -48, err
    assert nonfinite <= (1 << 22) // 1000
    err1, _ = gpu_ctx.selftest_alpha(1 << 22, 7, 1)
    assert err1 > err  # the refinement step is doing work


def test_cycle_fast_alpha_error_is_inside_the_analysed_bound(gpu_ctx):
    """The Form A fused kernels' rotation fast path (tsg_device.cuh, kGuardCycle): per triangle
    |t - alpha_ref/K| <= 9.5u (u = 2^-53) by the error analysis, so the decision band 2^-48 = 32u
    has a 1.66x margin over the worst-case difference of two minima (19.3u)."""
    u = 2.0 ** -53
    for seed in (11, 12, 13):
        err, nonfinite = gpu_ctx.selftest_alpha_cycle(1 << 22, seed)
        assert err <= 9.5 * u, err / u
        assert 2 * err + 0.3 * u <= 2.0 ** -48
        assert nonfinite <= (1 << 22) // 1000


FLOW_A_CASES = ["grid100_formA_tol0", "d10k_formA_tol0", "d10k_formA_serial_conv", "grid17x23_formA", "d300_formA",
                "d100k_formA_20"]


@pytest.mark.parametrize("layout,precision", [("aos", "f64"), ("soa", "f64")])
@pytest.mark.parametrize("name", FLOW_A_CASES)
def test_form_a_tile_flow_matches_golden(capi, gpu_ctx, ts, golden, monkeypatch, name, layout, precision):
    """Form A through the (tile, pass) dataflow kernel (tile_flow, TSG_FORMA_FLOW=1): the
    reference's digests bit for bit, including the displacement stop inside a 64-pass round
    (replayed from the round start) and the no-moves stop."""
    monkeypatch.setenv("TSG_FORMA_FLOW", "1")
    case = golden["cases"][name]
    xy, tri = fixture(ts, case["kind"], case["args"])
    kw = smooth_kwargs_to_capi(case["smooth"])
    dm, res = run_capi(capi, gpu_ctx, ts, xy, tri, kw["form"], kw["strategy"], kw["chunks"], kw["max_iters"],
                       kw["move_tol"], layout, reorder=True, precision=precision)
    assert res["schedule"] == "flow"
    assert_case(res, case)
    assert sha(dm.tri_alpha()) == case["tri_alpha"]
    dm.free()


@pytest.mark.parametrize("tile", ["768", "1024", "1280"])
def test_form_a_tile_flow_tile_sizes_and_copy_swap(capi, gpu_ctx, ts, golden, monkeypatch, tile):
    monkeypatch.setenv("TSG_FORMA_FLOW", "1")
    monkeypatch.setenv("TSG_TILE", tile)
    case = golden["cases"]["d100k_formA_20"]
    xy, tri = fixture(ts, case["kind"], case["args"])
    for swap in ("pingpong", "copy"):
        dm, res = run_capi(capi, gpu_ctx, ts, xy, tri, "a", max_iters=20, swap=swap, reorder=True)
        assert_case(res, case)
        dm.free()


def test_form_a_tile_flow_fp32_equals_graph(capi, gpu_ctx, ts, monkeypatch):
    """fp32: the dataflow launch and the per-pass graph give identical bits (same arithmetic,
    pass-start values only)."""
    xy, tri = ts.delaunay_arrays(200000, 9)
    out = {}
    for flow in ("0", "1"):
        monkeypatch.setenv("TSG_FORMA_FLOW", flow)
        dm, res = run_capi(capi, gpu_ctx, ts, xy, tri, "a", max_iters=40, move_tol=1e-7, reorder=True,
                           precision="f32")
        out[flow] = (res["iterations"], list(res["accepted"]), res["xy"].copy())
        dm.free()
    assert out["0"][0] == out["1"][0] and out["0"][1] == out["1"][1]
    assert np.array_equal(out["0"][2].view(np.uint64), out["1"][2].view(np.uint64))


def test_form_a_tile_flow_not_taken_with_side_rows(capi, gpu_ctx, ts, port, monkeypatch):
    """A mesh with rows of valence >= 32 keeps the per-pass graph (side_rows) under
    TSG_FORMA_FLOW=1, with the reference's results."""
    monkeypatch.setenv("TSG_FORMA_FLOW", "1")
    xy, tri = ts.graded_arrays(60000, 3, 2e-3, 2048)
    dm, res = run_capi(capi, gpu_ctx, ts, xy, tri, "a", max_iters=8, reorder=True)
    assert res["schedule"] == "graph"
    want = port.smooth(xy, tri, form="a", max_iters=8, move_tol=0.0)
    assert np.array_equal(res["xy"].view(np.uint64), want.xy.view(np.uint64))
    dm.free()
