"""The drop-in Python API on the GPU: the reference's smoke tests for smooth()
(proj/tests/python/test_smoke.py:35-59) plus full write-back parity of trismooth.smooth() —
coordinates, boundary flags, triangle alpha field, vertex minima and RunStats — against the
reference's golden outputs."""
import numpy as np
import pytest

import trismooth as ts
from helpers import sha

pytestmark = pytest.mark.gpu


def test_smooth_improves_quality():
    m = ts.generate_grid(20, 20, perturbation=0.3, seed=3)
    stats = ts.smooth(m, form="b", strategy="twophase", backend="serial")
    assert stats["iterations"] >= 1
    assert stats["stop"] in ("max_iters", "displacement", "no_moves")
    assert stats["mean_alpha_after"] > stats["mean_alpha_before"]
    assert stats["min_alpha_after"] >= stats["min_alpha_before"]
    assert len(stats["accepted_per_pass"]) == stats["iterations"]
    assert stats["total_ms"] >= stats["iter_ms"]


def test_smooth_keeps_boundary_fixed():
    m = ts.generate_grid(8, 8, perturbation=0.25, seed=11)
    before = m.points()
    boundary = m.boundary()
    ts.smooth(m, max_iters=5)
    after = m.points()
    flags = m.boundary()
    assert any(not f for f in flags)
    assert sum(1 for i in range(len(after)) if after[i] != before[i]) > 0
    for i, pinned in enumerate(flags):
        if pinned:
            assert after[i] == before[i]
    assert len(boundary) == len(flags)


@pytest.mark.parametrize("name", ["grid100_defaults", "d10k_formB_w8_soa_tol0", "d10k_formA_serial_conv",
                                  "d10k_formB_w3_fused", "grid12_formB_loose"])
@pytest.mark.parametrize("precision_layout", ["as_case", "other_layout"])
def test_drop_in_smooth_write_back(golden, name, precision_layout):
    case = golden["cases"][name]
    kw = dict(case["smooth"])
    layout = kw.pop("layout", "aos")
    if precision_layout == "other_layout":
        layout = "soa" if layout == "aos" else "aos"
    if case["kind"] == "grid":
        m = ts.generate_grid(*case["args"][:2], perturbation=case["args"][2], seed=case["args"][3], layout=layout)
    else:
        m = ts.generate_delaunay(case["args"][0], seed=case["args"][1], layout=layout)
    s = ts.smooth(m, **kw, detailed=True)
    assert s["iterations"] == case["iterations"] and s["stop"] == case["stop"]
    assert s["accepted_per_pass"] == case["accepted"]
    assert [float(x).hex() for x in s["max_disp_per_pass"]] == case["max_disp"]
    assert sha(m.points_array()) == case["xy_out"]
    assert sha(m.tri_alphas()) == case["tri_alpha"]
    assert sha(m.vertex_minima()) == case["vertex_min"]
    assert sha(np.array(m.boundary(), dtype=np.uint8)) == case["boundary"]
    for k in ("min_alpha_before", "min_alpha_after", "mean_alpha_before", "mean_alpha_after"):
        assert float(s[k]).hex() == case[k], k


def test_drop_in_formA_reorder_auto_on_large_mesh(golden):
    case = golden["cases"]["d100k_formA_20"]
    m = ts.generate_delaunay(100000, seed=42)
    s = ts.smooth(m, form="a", max_iters=20, move_tol=0.0, reorder="auto", detailed=True)
    assert s["accepted_per_pass"] == case["accepted"]
    assert sha(m.points_array()) == case["xy_out"]
    assert sha(m.vertex_minima()) == case["vertex_min"]


def test_f32_drop_in_runs_and_improves():
    m = ts.generate_delaunay(20000, seed=3)
    s = ts.smooth(m, form="a", precision="f32", max_iters=50, move_tol=0.0)
    assert s["mean_alpha_after"] > s["mean_alpha_before"]


def test_device_mesh_class_round_trip():
    xy, tri = ts.delaunay_arrays(5000, 9)
    topo = ts.topology(len(xy), tri)
    dm = ts.DeviceMesh(xy, tri, topo, "soa", "f64", True)
    assert np.array_equal(dm.get_coords(), xy)
    r = dm.run(ts.bbox_diagonal(xy), form="a", max_iters=10)
    assert r["iterations"] == 10 and len(r["max_disp_per_pass"]) == 10


@pytest.mark.parametrize("form,strategy,move_tol,forma_flow", [
    ("a", "fused", 1e-6, "1"),       # Form A dataflow forced, displacement stop live: rounds on the host
    ("a", "fused", 1e-6, None),      # AUTO: the per-pass graph (displacement stop live)
    ("a", "fused", 0.0, None),       # Form A dataflow, one launch, stop rule on the device
    ("a", "fused", 1e-6, "0"),       # Form A per-pass graph
    ("b", "twophase", 1e-6, None),   # serial Form B (reference defaults): formb_flow
])
def test_smooth_host_batch_equals_single_calls(capi, gpu_ctx, ts, port, monkeypatch, form, strategy, move_tol,
                                               forma_flow):
    """tsg_smooth_host_batch (copies overlapped with the passes, two staging slots) gives, item by
    item, exactly what tsg_smooth_host gives; odd and even item counts, different inputs; for
    every schedule the batch path can take."""
    if forma_flow is not None:
        monkeypatch.setenv("TSG_FORMA_FLOW", forma_flow)
    xy, tri = ts.delaunay_arrays(7000, 21)
    topo = ts.topology(len(xy), tri)
    dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo, order=capi.hilbert_order(xy))
    cfg = capi.make_cfg(form=form, strategy=strategy, max_iters=30, move_tol=move_tol,
                        bbox_diag=ts.bbox_diagonal(xy))
    rng = np.random.default_rng(3)
    ins = [np.ascontiguousarray(xy + rng.normal(0, 1e-4, xy.shape) * (k % 2)) for k in range(5)]
    for n in (1, 2, 5):
        outs = [np.empty_like(xy) for _ in range(n)]
        its, stops = dm.smooth_host_batch(ins[:n], cfg, outs)
        for k in range(n):
            want, r = dm.smooth_host(ins[k], cfg)
            assert its[k] == r["iterations"] and stops[k] == r["stop"]
            assert np.array_equal(outs[k].view(np.uint64), want.view(np.uint64))
    want = port.smooth(ins[0], tri, form=form, max_iters=30, move_tol=move_tol)
    outs = [np.empty_like(xy)]
    dm.smooth_host_batch(ins[:1], cfg, outs)
    assert np.array_equal(outs[0].view(np.uint64), want.xy.view(np.uint64))
    dm.free()


def test_smooth_host_batch_with_persistent_side_rows(capi, gpu_ctx, ts, port):
    """The batch path (graph driver) with the high-valence rows in the persistent side kernel:
    every item equals the reference (the side kernel's ticket counter is reused across items)."""
    xy, tri = ts.graded_arrays(30000, 5, 2e-3, 600)
    topo = ts.topology(len(xy), tri)
    assert np.diff(topo["nbr_off"]).max() > 256
    dm = capi.DeviceMesh(gpu_ctx, xy, tri, topo, order=capi.hilbert_order(xy))
    dm.side_schedule("persist")
    cfg = capi.make_cfg(form="a", max_iters=12, move_tol=0.0, bbox_diag=ts.bbox_diagonal(xy))
    rng = np.random.default_rng(5)
    ins = [np.ascontiguousarray(xy + rng.normal(0, 1e-5, xy.shape) * k) for k in range(3)]
    outs = [np.empty_like(xy) for _ in ins]
    dm.smooth_host_batch(ins, cfg, outs)
    for k in range(3):
        want = port.smooth(ins[k], tri, form="a", max_iters=12, move_tol=0.0)
        assert np.array_equal(outs[k].view(np.uint64), want.xy.view(np.uint64)), k
    dm.free()


def test_upload_rejects_malformed_descriptions(capi, gpu_ctx, ts):
    """tsg_mesh_upload validates caller arrays before indexing through them (the reference's
    build_mesh raises StructuralError on bad corner ids, proj/src/mesh.cpp:69-81)."""
    xy, tri = ts.delaunay_arrays(500, 1)
    topo = ts.topology(len(xy), tri)

    def upload(tri_=tri, **over):
        t = {k: np.array(v, copy=True) for k, v in topo.items()}
        t.update(over)
        return capi.DeviceMesh(gpu_ctx, xy, tri_, t)

    bad_tri = tri.copy()
    bad_tri[3, 1] = len(xy)
    with pytest.raises(RuntimeError, match="corner index out of range"):
        upload(bad_tri)
    nbr = topo["nbr"].copy()
    r = int(np.argmax(np.diff(topo["nbr_off"]) > 2))
    a = int(topo["nbr_off"][r])
    nbr[a], nbr[a + 1] = nbr[a + 1], nbr[a]
    with pytest.raises(RuntimeError, match="neighbour CSR malformed"):
        upload(nbr=nbr)
    inc = topo["inc"].copy()
    inc[7] = len(tri) + 3
    with pytest.raises(RuntimeError, match="incident CSR malformed"):
        upload(inc=inc)
    off = topo["inc_off"].copy()
    off[10] = off[12]
    with pytest.raises(RuntimeError, match="incident CSR malformed"):
        upload(inc_off=off)
    upload().free()  # the untouched description still uploads


_CONCURRENT_SCRIPT = r"""
import sys, threading
sys.path.insert(0, sys.argv[1])
import paper_1502_00355_b200 as ts
seeds = [3, 4, 5, 6]
want = []
for s in seeds:
    m = ts.generate_delaunay(8000, seed=s)
    ts.smooth(m, form="a", max_iters=20, move_tol=0.0)
    want.append(m.points())
for rep in range(3):
    meshes = [ts.generate_delaunay(8000, seed=s) for s in seeds]
    errors = []
    def work(m):
        try:
            ts.smooth(m, form="a", max_iters=20, move_tol=0.0)
        except Exception as exc:
            errors.append(exc)
    threads = [threading.Thread(target=work, args=(m,)) for m in meshes]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for m, w in zip(meshes, want):
        assert m.points() == w
print("ok")
"""


def test_concurrent_smooth_calls_share_the_default_context():
    """The drop-in smooth() shares one process-wide device context; concurrent calls on
    distinct meshes from several host threads (the GIL is released) give the sequential
    results (tsg_context::mu serialises the C-ABI calls).  Runs in a child process with
    TSG_SEGV_TRACE=1 so that a crash is reported with its native stack instead of ending the
    test session."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TSG_SEGV_TRACE="1")
    r = subprocess.run([sys.executable, "-c", _CONCURRENT_SCRIPT, root], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (r.returncode, r.stdout[-2000:], r.stderr[-6000:])
