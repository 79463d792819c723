"""Generates the committed golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run here (where /root/reference exists):  python tests/golden/make_golden.py [--big]

It loads oracle/_ref/libtsref.so — the reference's own sources (/root/reference/proj/src)
compiled out-of-tree by oracle/Makefile — and records, for a set of seeded synthetic meshes
and smoothing configurations, the reference's outputs:

* golden.json  pinned values (alpha, SplitMix64 streams), and for every case the iteration
  count, stop reason, accepted_per_pass, max_disp_per_pass (float64 hex), min/mean alpha
  before/after, and sha256 digests of the final coordinates, triangle alpha field and vertex
  minima (little-endian float64 bytes in original order) plus of the input triangles;
* small_cases.npz  full input/output arrays of the small cases, so tests can report the
  first differing vertex instead of a digest mismatch.

With --big it also pins the 1M-point Delaunay fixture (reference generator, ~150 s) and 10
Form A passes on it.  Nothing in tests/ reads /root/reference at run time.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Ref  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<"), copy=False).tobytes()).hexdigest()


def hexlist(a) -> list[str]:
    return [float(x).hex() for x in a]


# (name, generator, generator args, smooth kwargs)
CASES = [
    # cfg1 as-is: SmoothConfig{} defaults (Form B, TwoPhase, Serial, 100, 1e-6), AoS
    ("grid100_defaults", "grid", (100, 100, 0.3, 1), dict()),
    ("grid100_formA_tol0", "grid", (100, 100, 0.3, 1), dict(form="a", max_iters=100, move_tol=0.0)),
    ("d10k_formA_tol0", "delaunay", (10000, 42), dict(form="a", max_iters=100, move_tol=0.0)),
    ("d10k_formB_w8_soa_tol0", "delaunay", (10000, 42),
     dict(form="b", backend="parallel", workers=8, layout="soa", max_iters=100, move_tol=0.0)),
    ("d10k_formB_serial_conv", "delaunay", (10000, 42), dict(form="b", max_iters=1000, move_tol=1e-6)),
    ("d10k_formA_serial_conv", "delaunay", (10000, 42), dict(form="a", max_iters=1000, move_tol=1e-6)),
    ("d10k_formB_w3_fused", "delaunay", (10000, 42),
     dict(form="b", strategy="fused", backend="parallel", workers=3, max_iters=50, move_tol=0.0)),
    ("d1k_formB_w148", "delaunay", (1000, 1000),
     dict(form="b", backend="parallel", workers=148, max_iters=30, move_tol=0.0)),
    ("grid17x23_formA", "grid", (17, 23, 0.3, 42), dict(form="a", max_iters=50, move_tol=1e-6)),
    ("grid12_formB_loose", "grid", (12, 12, 0.3, 3), dict(form="b", max_iters=100, move_tol=1e-3)),
    ("d300_formA", "delaunay", (300, 77), dict(form="a", max_iters=30, move_tol=1e-6)),
    ("d100k_formA_20", "delaunay", (100000, 42), dict(form="a", max_iters=20, move_tol=0.0)),
]
SMALL = {"grid17x23_formA", "grid12_formB_loose", "d300_formA", "d1k_formB_w148"}


def make_mesh(ref: Ref, kind, args):
    if kind == "grid":
        return ref.perturbed_grid(*args)
    n, seed = args
    return ref.delaunay(n, seed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    opt = ap.parse_args()
    ref = Ref()
    out = {
        "generator": "tests/golden/make_golden.py (reference compiled from /root/reference/proj/src)",
        "hash": "sha256 over little-endian float64 / int32 arrays in original order",
        "alpha_pinned": {
            "equilateral": ref.alpha((0, 0), (1, 0), (0.5, 3 ** 0.5 / 2)).hex(),
            "right_isoceles": ref.alpha((0, 0), (1, 0), (0, 1)).hex(),
            "collinear": ref.alpha((0, 0), (1, 0), (2, 0)).hex(),
            "reversed": ref.alpha((0, 0), (0, 1), (1, 0)).hex(),
            "coincident": ref.alpha((4, 4), (4, 4), (4, 4)).hex(),
        },
        "splitmix": {"0": [f"{x:016x}" for x in ref.splitmix(0, 3)],
                     "1234567": [f"{x:016x}" for x in ref.splitmix(1234567, 2)]},
        "cases": {},
    }
    arrays = {}
    cases = list(CASES)
    if opt.big:
        cases.append(("d1m_formA_10", "delaunay", (1000000, 42), dict(form="a", max_iters=10, move_tol=0.0)))
    for name, kind, args, kw in cases:
        t0 = time.time()
        xy, tri = make_mesh(ref, kind, args)
        r = ref.smooth(xy, tri, **kw)
        topo = ref.topology(xy, tri)
        rec = dict(kind=kind, args=list(args), smooth=kw, nv=len(xy), nt=len(tri),
                   xy_in=sha(xy), tri=sha(tri), boundary=sha(topo["boundary"]),
                   n_boundary=int(topo["boundary"].sum()),
                   iterations=r.iterations, stop=r.stop, accepted=[int(a) for a in r.accepted],
                   max_disp=hexlist(r.max_disp), xy_out=sha(r.xy), tri_alpha=sha(r.tri_alpha),
                   vertex_min=sha(r.vertex_min),
                   min_alpha_before=r.stats["min_alpha_before"].hex(),
                   min_alpha_after=r.stats["min_alpha_after"].hex(),
                   mean_alpha_before=r.stats["mean_alpha_before"].hex(),
                   mean_alpha_after=r.stats["mean_alpha_after"].hex(),
                   accepted_total=int(r.accepted.sum()))
        out["cases"][name] = rec
        if name in SMALL:
            arrays[f"{name}__xy"] = xy
            arrays[f"{name}__tri"] = tri
            arrays[f"{name}__xy_out"] = r.xy
        print(f"{name}: {r.iterations} iters ({r.stop}), accepted {rec['accepted_total']} [{time.time() - t0:.1f}s]",
              flush=True)
    path = os.path.join(HERE, "golden.json" if not opt.big else "golden_big.json")
    with open(path, "w") as f:
        json.dump(out if not opt.big else {k: v for k, v in out["cases"].items() if k.startswith("d1m")},
                  f, indent=1, sort_keys=True)
    if not opt.big:
        np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    print("wrote", path)


if __name__ == "__main__":
    main()
