"""ctypes face of the TEST-ONLY checkers in oracle/.

THIS IS TEST INFRASTRUCTURE.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the checker or
the timed CPU baseline — never as the thing measured or shipped.

Two checkers:

* ``Ref``  — the reference library itself (``/root/reference/proj/src/*.cpp``) compiled
  out-of-tree by ``oracle/Makefile`` into ``oracle/_ref/libtsref.so`` (see ref_shim.cpp).
* ``Port`` — the plain-C restatement ``oracle/smart_laplacian.c`` → ``oracle/liboracle.so``.

Both take / return numpy arrays: ``xy`` float64 (nv, 2), ``tri`` int32 (nt, 3).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libtsref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")

_P = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_u64 = C.c_uint64
_dbl = C.c_double

STOP_NAMES = ("max_iters", "displacement", "no_moves")


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class SmoothResult:
    xy: np.ndarray
    accepted: np.ndarray
    max_disp: np.ndarray
    iterations: int
    stop: str
    boundary: np.ndarray | None = None
    tri_alpha: np.ndarray | None = None
    vertex_min: np.ndarray | None = None
    stats: dict = field(default_factory=dict)


def fnv1a64_coords(xy: np.ndarray) -> str:
    """FNV-1a-64 over raw little-endian doubles (x, y) per vertex."""
    data = np.ascontiguousarray(xy, dtype="<f8")
    lib = C.CDLL(PORT_SO)
    lib.orc_fnv1a64.restype = _u64
    lib.orc_fnv1a64.argtypes = [_P, _i64]
    return f"{lib.orc_fnv1a64(_ptr(data), data.nbytes):016x}"


class Ref:
    """The reference itself (compiled from /root/reference sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.tsref_last_error.restype = C.c_char_p
        L.tsref_hardware_concurrency.restype = C.c_uint
        L.tsref_triangle_alpha.restype = _dbl
        L.tsref_triangle_alpha.argtypes = [_dbl] * 6
        L.tsref_splitmix_stream.argtypes = [_u64, C.c_int, _P]
        L.tsref_perturbed_grid.argtypes = [C.c_int, C.c_int, _dbl, _u64, _P, _P]
        L.tsref_generate_points.argtypes = [C.c_int, _u64, _P]
        L.tsref_triangulate.restype = _i64
        L.tsref_triangulate.argtypes = [_P, _i64, _P, _i64]
        L.tsref_text_hashes.argtypes = [_P, _i64, _P, _i64, _P, _P]
        L.tsref_topology.argtypes = [_P, _i64, _P, _i64] + [_P] * 6
        L.tsref_smooth.argtypes = [_P, _i64, _P, _i64, _P, _dbl, _P, _P, _P, _P, _i32, _P, _P, _P]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.tsref_last_error().decode())

    def hardware_concurrency(self) -> int:
        return int(self.lib.tsref_hardware_concurrency())

    def alpha(self, p1, p2, p3) -> float:
        return self.lib.tsref_triangle_alpha(*p1, *p2, *p3)

    def splitmix(self, seed: int, count: int) -> list[int]:
        out = np.zeros(count, dtype=np.uint64)
        self.lib.tsref_splitmix_stream(seed, count, _ptr(out))
        return [int(x) for x in out]

    def perturbed_grid(self, rows, cols, pert=0.3, seed=1):
        xy = np.zeros((rows * cols, 2))
        tri = np.zeros((2 * (rows - 1) * (cols - 1), 3), dtype=np.int32)
        self._check(self.lib.tsref_perturbed_grid(rows, cols, pert, seed, _ptr(xy), _ptr(tri)))
        return xy, tri

    def generate_points(self, n, seed):
        xy = np.zeros((n, 2))
        self._check(self.lib.tsref_generate_points(n, seed, _ptr(xy)))
        return xy

    def triangulate(self, xy):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        cap = 2 * len(xy) + 8
        tri = np.zeros((cap, 3), dtype=np.int32)
        nt = self.lib.tsref_triangulate(_ptr(xy), len(xy), _ptr(tri), cap)
        if nt < 0:
            raise RuntimeError(self.lib.tsref_last_error().decode())
        return tri[:nt].copy()

    def delaunay(self, n, seed):
        xy = self.generate_points(n, seed)
        return xy, self.triangulate(xy)

    def text_hashes(self, xy, tri):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        a, b = _u64(), _u64()
        self._check(self.lib.tsref_text_hashes(_ptr(xy), len(xy), _ptr(tri), len(tri), C.byref(a), C.byref(b)))
        return f"{a.value:016x}", f"{b.value:016x}"

    def topology(self, xy, tri):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        nv, nt = len(xy), len(tri)
        nbr_off = np.zeros(nv + 1, dtype=np.int64)
        inc_off = np.zeros(nv + 1, dtype=np.int64)
        nbr = np.zeros(6 * nt, dtype=np.int32)
        mult = np.zeros(6 * nt, dtype=np.int32)
        inc = np.zeros(3 * nt, dtype=np.int32)
        bnd = np.zeros(nv, dtype=np.uint8)
        self._check(self.lib.tsref_topology(_ptr(xy), nv, _ptr(tri), nt, _ptr(nbr_off), _ptr(nbr),
                                            _ptr(mult), _ptr(inc_off), _ptr(inc), _ptr(bnd)))
        m = int(nbr_off[-1])
        return dict(nbr_off=nbr_off, nbr=nbr[:m], mult=mult[:m], inc_off=inc_off,
                    inc=inc[: int(inc_off[-1])], boundary=bnd)

    def smooth(self, xy, tri, form="b", strategy="twophase", backend="serial", workers=1,
               max_iters=100, move_tol=1e-6, layout="aos") -> SmoothResult:
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        nv, nt = len(xy), len(tri)
        cfg = np.array([0 if layout == "aos" else 1, 0 if form == "a" else 1,
                        0 if strategy == "fused" else 1, 0 if backend == "serial" else 1,
                        workers, max_iters], dtype=np.int32)
        out = np.zeros_like(xy)
        bnd = np.zeros(nv, dtype=np.uint8)
        acc = np.zeros(max_iters, dtype=np.int32)
        md = np.zeros(max_iters)
        st = np.zeros(11)
        alpha = np.zeros(nt)
        vmin = np.zeros(nv)
        self._check(self.lib.tsref_smooth(_ptr(xy), nv, _ptr(tri), nt, _ptr(cfg), move_tol, _ptr(out),
                                          _ptr(bnd), _ptr(acc), _ptr(md), max_iters, _ptr(st),
                                          _ptr(alpha), _ptr(vmin)))
        it = int(st[0])
        keys = ("iterations", "stop", "init_ms", "topo_ms", "constr_ms", "iter_ms", "total_ms",
                "min_alpha_before", "min_alpha_after", "mean_alpha_before", "mean_alpha_after")
        stats = dict(zip(keys, st.tolist()))
        stats["iterations"] = it
        stats["stop"] = STOP_NAMES[int(st[1])]
        return SmoothResult(out, acc[:it].copy(), md[:it].copy(), it, STOP_NAMES[int(st[1])], bnd,
                            alpha, vmin, stats)


class Port:
    """The plain-C restatement (oracle/smart_laplacian.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        L.orc_alpha.restype = _dbl
        L.orc_alpha.argtypes = [_dbl] * 6
        L.orc_splitmix_next.restype = _u64
        L.orc_splitmix_next.argtypes = [_P]
        L.orc_perturbed_grid.argtypes = [C.c_int, C.c_int, _dbl, _u64, _P, _P]
        L.orc_topology.argtypes = [_i64, _i64, _P] + [_P] * 6
        L.orc_smooth.argtypes = [_i64, _i64, _P, _P, C.c_int, _i64, C.c_int, _dbl, _P, _P, C.c_int,
                                 _P, _P, _P, _P]
        L.orc_smooth_prepared.argtypes = [_i64, _i64] + [_P] * 7 + [C.c_int, _i64, C.c_int, _dbl,
                                                                    _P, _P, C.c_int, _P, _P, _P]
        L.orc_pass_lockstep.argtypes = [_i64, _i64] + [_P] * 7 + [C.c_int, _i64, C.c_int, _P, _P, _P]
        L.orc_lockstep_sample.argtypes = [_P] * 8 + [_i64, C.c_int, _P, _P, _P]

    def alpha(self, p1, p2, p3) -> float:
        return self.lib.orc_alpha(*p1, *p2, *p3)

    def splitmix(self, seed: int, count: int) -> list[int]:
        s = np.array([seed], dtype=np.uint64)
        return [int(self.lib.orc_splitmix_next(_ptr(s))) for _ in range(count)]

    def perturbed_grid(self, rows, cols, pert=0.3, seed=1):
        xy = np.zeros((rows * cols, 2))
        tri = np.zeros((2 * (rows - 1) * (cols - 1), 3), dtype=np.int32)
        if self.lib.orc_perturbed_grid(rows, cols, pert, seed, _ptr(xy), _ptr(tri)):
            raise RuntimeError("invalid grid spec")
        return xy, tri

    def topology(self, nv, tri):
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        nt = len(tri)
        nbr_off = np.zeros(nv + 1, dtype=np.int64)
        inc_off = np.zeros(nv + 1, dtype=np.int64)
        nbr = np.zeros(6 * nt + 1, dtype=np.int32)
        mult = np.zeros(6 * nt + 1, dtype=np.int32)
        inc = np.zeros(3 * nt + 1, dtype=np.int32)
        bnd = np.zeros(nv, dtype=np.uint8)
        if self.lib.orc_topology(nv, nt, _ptr(tri), _ptr(nbr_off), _ptr(nbr), _ptr(mult),
                                 _ptr(inc_off), _ptr(inc), _ptr(bnd)):
            raise MemoryError("orc_topology")
        m = int(nbr_off[-1])
        return dict(nbr_off=nbr_off, nbr=nbr[:m].copy(), mult=mult[:m].copy(), inc_off=inc_off,
                    inc=inc[: int(inc_off[-1])].copy(), boundary=bnd)

    def smooth(self, xy, tri, form="a", chunks=1, max_iters=100, move_tol=1e-6) -> SmoothResult:
        """form 'a'|'b'; chunks = 1 (serial) or W (reference Backend::Parallel, W workers)."""
        xy = np.array(xy, dtype=np.float64, order="C", copy=True)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        nv, nt = len(xy), len(tri)
        acc = np.zeros(max_iters, dtype=np.int32)
        md = np.zeros(max_iters)
        st = np.zeros(6)
        bnd = np.zeros(nv, dtype=np.uint8)
        alpha = np.zeros(nt)
        vmin = np.zeros(nv)
        if self.lib.orc_smooth(nv, nt, _ptr(tri), _ptr(xy), 0 if form == "a" else 1, chunks, max_iters,
                               move_tol, _ptr(acc), _ptr(md), max_iters, _ptr(st), _ptr(bnd),
                               _ptr(alpha), _ptr(vmin)):
            raise MemoryError("orc_smooth")
        it = int(st[0])
        stats = dict(iterations=it, stop=STOP_NAMES[int(st[1])], min_alpha_before=st[2],
                     min_alpha_after=st[3], mean_alpha_before=st[4], mean_alpha_after=st[5])
        return SmoothResult(xy, acc[:it].copy(), md[:it].copy(), it, STOP_NAMES[int(st[1])], bnd,
                            alpha, vmin, stats)

    def smooth_prepared(self, topo, tri, xy, form="a", chunks=1, max_iters=100, move_tol=0.0):
        xy = np.array(xy, dtype=np.float64, order="C", copy=True)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        nv, nt = len(xy), len(tri)
        acc = np.zeros(max_iters, dtype=np.int32)
        md = np.zeros(max_iters)
        st = np.zeros(6)
        if self.lib.orc_smooth_prepared(nv, nt, _ptr(tri), _ptr(topo["nbr_off"]), _ptr(topo["nbr"]),
                                        _ptr(topo["inc_off"]), _ptr(topo["inc"]), _ptr(topo["boundary"]),
                                        _ptr(xy), 0 if form == "a" else 1, chunks, max_iters, move_tol,
                                        _ptr(acc), _ptr(md), max_iters, _ptr(st), None, None):
            raise MemoryError("orc_smooth_prepared")
        it = int(st[0])
        return SmoothResult(xy, acc[:it].copy(), md[:it].copy(), it, STOP_NAMES[int(st[1])])

    def lockstep_sample(self, topo, tri, xy, ids, precision=0):
        """Form A lockstep pass evaluated only at `ids` (orc_lockstep_sample): (new positions of
        ids, decisions, f64 margins)."""
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.zeros((len(ids), 2))
        dec = np.zeros(len(ids), dtype=np.int8)
        margin = np.zeros(len(ids))
        self.lib.orc_lockstep_sample(_ptr(tri), _ptr(topo["nbr_off"]), _ptr(topo["nbr"]), _ptr(topo["inc_off"]),
                                     _ptr(topo["inc"]), _ptr(topo["boundary"]), _ptr(xy), _ptr(ids), len(ids),
                                     precision, _ptr(out), _ptr(dec), _ptr(margin))
        return out, dec, margin

    def pass_lockstep(self, topo, tri, xy, form="a", chunks=1, precision=0):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        nv, nt = len(xy), len(tri)
        out = np.zeros_like(xy)
        dec = np.zeros(nv, dtype=np.int8)
        margin = np.zeros(nv)
        self.lib.orc_pass_lockstep(nv, nt, _ptr(tri), _ptr(topo["nbr_off"]), _ptr(topo["nbr"]),
                                   _ptr(topo["inc_off"]), _ptr(topo["inc"]), _ptr(topo["boundary"]),
                                   _ptr(xy), 0 if form == "a" else 1, chunks, precision, _ptr(out),
                                   _ptr(dec), _ptr(margin))
        return out, dec, margin
