"""Shared helpers for the parity tests (mesh fixtures from the product generators)."""
import hashlib

import numpy as np


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<"), copy=False).tobytes()).hexdigest()


def fixture(ts, kind, args):
    """Mesh arrays from the product's generators (pinned to the reference by test_host_api)."""
    if kind == "grid":
        return ts.grid_arrays(*args)
    n, seed = args
    return ts.delaunay_arrays(n, seed)


def smooth_kwargs_to_capi(kw):
    """Reference smooth() keyword arguments -> (form, strategy, chunks, max_iters, move_tol, layout)."""
    form = kw.get("form", "b")
    strategy = kw.get("strategy", "twophase")
    chunks = kw.get("workers", 1) if kw.get("backend", "serial") == "parallel" else 1
    return dict(form=form, strategy=strategy, chunks=chunks, max_iters=kw.get("max_iters", 100),
                move_tol=kw.get("move_tol", 1e-6), layout=kw.get("layout", "aos"))


def fan(n, center):
    pts = [center] + [(np.cos(2 * np.pi * k / n), np.sin(2 * np.pi * k / n)) for k in range(n)]
    tris = [(0, 1 + k, 1 + (k + 1) % n) for k in range(n)]
    return np.array(pts, dtype=np.float64), np.array(tris, dtype=np.int32)
