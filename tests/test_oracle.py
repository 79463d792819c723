"""The oracle is pinned before it is trusted (CPU only).

* the plain-C restatement (oracle/liboracle.so) reproduces every committed golden case,
  which were generated from the reference itself (tests/golden/make_golden.py);
* when the reference build is present (this container), restatement == reference on fresh
  seeds across forms, chunk counts and stop rules;
* the known-answer values of the reference's own tests (alpha pinned values,
  proj/tests/test_quality.cpp:37-43; SplitMix64 streams, proj/tests/test_meshgen.cpp:25-33)
  and the survey's Σaccepted figures (G1..G6).
"""
import math

import numpy as np
import pytest

from helpers import fixture, sha, smooth_kwargs_to_capi

SURVEY_ACCEPTED = {  # SURVEY.md Appendix B, "Golden" table
    "grid100_defaults": (100, 451243),
    "grid100_formA_tol0": (100, 480779),
    "d10k_formA_tol0": (100, 115176),
    "d10k_formB_w8_soa_tol0": (100, 113755),
    "d10k_formB_serial_conv": (42, 115124),
    "d10k_formA_serial_conv": (63, 106209),
}


def test_alpha_known_answers(port, golden):
    r3 = math.sqrt(3) / 2
    assert abs(port.alpha((0, 0), (1, 0), (0.5, r3)) - 1.0) <= 1e-6
    assert port.alpha((0, 0), (1, 0), (2, 0)) == 0.0
    assert abs(port.alpha((0, 0), (1, 0), (0, 1)) - r3) <= 1e-6
    assert abs(port.alpha((0, 0), (0, 1), (1, 0)) + 0.8660254) <= 1e-6
    assert port.alpha((3, 7), (3, 7), (3, 7)) == 0.0
    pinned = golden["alpha_pinned"]
    assert port.alpha((0, 0), (1, 0), (0.5, 3 ** 0.5 / 2)).hex() == pinned["equilateral"]
    assert port.alpha((0, 0), (1, 0), (0, 1)).hex() == pinned["right_isoceles"]
    assert port.alpha((0, 0), (0, 1), (1, 0)).hex() == pinned["reversed"]


def test_splitmix_known_answers(port, golden):
    assert port.splitmix(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert port.splitmix(1234567, 2) == [0x599ED017FB08FC85, 0x2C73F08458540FA5]
    assert [f"{x:016x}" for x in port.splitmix(0, 3)] == golden["splitmix"]["0"]


def test_survey_accepted_totals(golden):
    for name, (iters, total) in SURVEY_ACCEPTED.items():
        case = golden["cases"][name]
        assert case["iterations"] == iters and case["accepted_total"] == total, name


@pytest.mark.parametrize("name", [
    "grid100_defaults", "grid100_formA_tol0", "d10k_formA_tol0", "d10k_formB_w8_soa_tol0",
    "d10k_formB_serial_conv", "d10k_formA_serial_conv", "d10k_formB_w3_fused", "d1k_formB_w148",
    "grid17x23_formA", "grid12_formB_loose", "d300_formA"])
def test_port_reproduces_golden(port, ts, golden, name):
    case = golden["cases"][name]
    xy, tri = fixture(ts, case["kind"], case["args"])
    assert sha(xy) == case["xy_in"] and sha(tri) == case["tri"]
    kw = smooth_kwargs_to_capi(case["smooth"])
    r = port.smooth(xy, tri, form=kw["form"], chunks=kw["chunks"], max_iters=kw["max_iters"],
                    move_tol=kw["move_tol"])
    assert r.iterations == case["iterations"] and r.stop == case["stop"]
    assert [int(a) for a in r.accepted] == case["accepted"]
    assert [float(x).hex() for x in r.max_disp] == case["max_disp"]
    assert sha(r.xy) == case["xy_out"]
    assert sha(r.tri_alpha) == case["tri_alpha"]
    assert sha(r.vertex_min) == case["vertex_min"]
    assert r.stats["mean_alpha_after"].hex() == case["mean_alpha_after"]
    assert sha(r.boundary) == case["boundary"]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_matches_reference_random(port, ref, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(200, 3000))
    xy, tri = ref.delaunay(n, seed + 100)
    for form in ("a", "b"):
        for workers in (1, 2, 7, 64):
            backend = "serial" if workers == 1 else "parallel"
            a = ref.smooth(xy, tri, form=form, backend=backend, workers=workers, max_iters=25, move_tol=1e-7)
            b = port.smooth(xy, tri, form=form, chunks=workers, max_iters=25, move_tol=1e-7)
            assert a.iterations == b.iterations and a.stop == b.stop
            assert np.array_equal(a.accepted, b.accepted)
            assert np.array_equal(a.max_disp.view(np.uint64), b.max_disp.view(np.uint64))
            assert np.array_equal(a.xy.view(np.uint64), b.xy.view(np.uint64)), (form, workers)


def test_port_topology_matches_reference(port, ref):
    for xy, tri in (ref.perturbed_grid(9, 13, 0.3, 5), ref.delaunay(777, 9)):
        a = ref.topology(xy, tri)
        b = port.topology(len(xy), tri)
        for k in ("nbr_off", "nbr", "mult", "inc_off", "inc", "boundary"):
            assert np.array_equal(a[k], b[k]), k


def test_lockstep_f64_equals_one_pass(port, ts):
    xy, tri = ts.delaunay_arrays(2000, 3)
    topo = port.topology(len(xy), tri)
    for form, chunks in (("a", 1), ("b", 1), ("b", 5)):
        out, dec, margin = port.pass_lockstep(topo, tri, xy, form=form, chunks=chunks, precision=0)
        r = port.smooth(xy, tri, form=form, chunks=chunks, max_iters=1, move_tol=0.0)
        assert np.array_equal(out.view(np.uint64), r.xy.view(np.uint64))
        assert int((dec == 1).sum()) == int(r.accepted[0])


@pytest.mark.parametrize("precision", [0, 1])
def test_lockstep_sample_equals_full_lockstep(port, ts, precision):
    """The sampled Form A lockstep (cfg5 parity) equals the full lockstep pass at
    the sampled vertices."""
    xy, tri = ts.delaunay_arrays(20000, 8)
    topo = port.topology(len(xy), tri)
    full, dec, margin = port.pass_lockstep(topo, tri, xy, form="a", precision=precision)
    ids = np.sort(np.random.default_rng(1).choice(len(xy), 3000, replace=False))
    out, sdec, smargin = port.lockstep_sample(topo, tri, xy, ids, precision=precision)
    assert np.array_equal(sdec, dec[ids])
    assert np.array_equal(smargin, margin[ids])
    assert np.array_equal(out.view(np.uint64), full[ids].view(np.uint64))
