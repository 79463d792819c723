"""ctypes binding of the C ABI in include/tsg.h (libtsg.so).

This is the binding a reference-side maintainer would add for the FFI route (see
INTEGRATION.md); the tests use it to exercise the C ABI directly and bench.py uses it for the
end-to-end (host buffers in, host buffers out) measurement.  It raises if libtsg.so is missing
or a call fails — no fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSG_LIB") or os.path.join(HERE, "libtsg.so")  # TSG_LIB: experiment builds

TSG_OK, TSG_ERR_INVALID, TSG_ERR_CUDA, TSG_ERR_NOMEM, TSG_ERR_NODEVICE = 0, 1, 2, 3, 4
LAYOUT = {"aos": 0, "soa": 1}
PRECISION = {"f64": 0, "f32": 1}
FORM = {"a": 0, "b": 1}
STRATEGY = {"fused": 0, "twophase": 1}
SWAP = {"pingpong": 0, "copy": 1}
DRIVER = {"graph": 0, "stream": 1}
STOP = ("max_iters", "displacement", "no_moves")

# Every symbol include/tsg.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "tsg_abi_version", "tsg_last_error", "tsg_device_count", "tsg_context_create",
    "tsg_context_destroy", "tsg_context_stream", "tsg_mesh_upload", "tsg_mesh_upload_triangles", "tsg_mesh_free",
    "tsg_mesh_device_bytes", "tsg_mesh_set_coords", "tsg_mesh_get_coords", "tsg_mesh_restore_coords",
    "tsg_tri_alpha",
    "tsg_vertex_minima", "tsg_alpha_extrema", "tsg_smooth", "tsg_smooth_host",
    "tsg_pass_lockstep", "tsg_smooth_host_batch", "tsg_hilbert_order", "tsg_selftest_alpha", "tsg_selftest_alpha_cycle", "tsg_pass", "tsg_halo_plan",
    "tsg_halo_pack", "tsg_halo_unpack", "tsg_dist_begin", "tsg_dist_pass", "tsg_dist_halo_pack",
    "tsg_dist_halo_unpack", "tsg_dist_finalize", "tsg_dist_status", "tsg_dist_end", "tsg_mesh_formb_schedule",
    "tsg_debug_trace", "tsg_mesh_side_schedule", "tsg_quality_tri_alpha", "tsg_quality_vertex_minima",
    "tsg_peer_local", "tsg_mesh_slots", "tsg_peer_setup", "tsg_peer_prepare", "tsg_peer_clear", "tsg_ipc_handle", "tsg_ipc_open",
    "tsg_ipc_close", "tsg_topology", "tsg_debug_layout_check", "tsg_hilbert_order_device",
)
IPC_HANDLE_BYTES = 64


class MeshDesc(C.Structure):
    _fields_ = [("nv", C.c_int64), ("nt", C.c_int64), ("xy", C.c_void_p), ("tri", C.c_void_p),
                ("nbr_off", C.c_void_p), ("nbr", C.c_void_p), ("inc_off", C.c_void_p),
                ("inc", C.c_void_p), ("boundary", C.c_void_p), ("order", C.c_void_p),
                ("layout", C.c_int32), ("precision", C.c_int32)]


class SmoothCfg(C.Structure):
    _fields_ = [("form", C.c_int32), ("strategy", C.c_int32), ("chunks", C.c_int32),
                ("swap", C.c_int32), ("max_iters", C.c_int32), ("driver", C.c_int32),
                ("move_tol", C.c_double), ("bbox_diag", C.c_double)]


QUALITY_BINS = 20


class QualityReport(C.Structure):
    _fields_ = [("min_alpha", C.c_double), ("max_alpha", C.c_double), ("non_positive", C.c_int64),
                ("histogram", C.c_int64 * QUALITY_BINS)]


class SmoothStats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("stop", C.c_int32), ("node_updates", C.c_int64),
                ("device_ms", C.c_double), ("node_kernel_ms", C.c_double), ("launches", C.c_int64),
                ("schedule", C.c_int32), ("reserved", C.c_int32)]


SCHEDULE = {0: "graph", 1: "stream", 2: "peer", 3: "flow"}


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing — build with `make` (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        P, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "tsg_abi_version": (i32, []),
            "tsg_last_error": (C.c_char_p, []),
            "tsg_device_count": (i32, []),
            "tsg_context_create": (i32, [i32, C.POINTER(P)]),
            "tsg_context_destroy": (i32, [P]),
            "tsg_context_stream": (P, [P]),
            "tsg_mesh_upload": (i32, [P, C.POINTER(MeshDesc), C.POINTER(P)]),
            "tsg_mesh_upload_triangles": (i32, [P, C.POINTER(MeshDesc), C.POINTER(P)]),
            "tsg_mesh_free": (i32, [P]),
            "tsg_mesh_device_bytes": (i64, [P]),
            "tsg_mesh_set_coords": (i32, [P, P]),
            "tsg_mesh_get_coords": (i32, [P, P]),
            "tsg_mesh_restore_coords": (i32, [P]),
            "tsg_tri_alpha": (i32, [P, P]),
            "tsg_vertex_minima": (i32, [P, P]),
            "tsg_alpha_extrema": (i32, [P, P, P, P]),
            "tsg_smooth": (i32, [P, C.POINTER(SmoothCfg), C.POINTER(SmoothStats), P, P, i32]),
            "tsg_smooth_host": (i32, [P, P, C.POINTER(SmoothCfg), P, C.POINTER(SmoothStats), P, P, i32]),
            "tsg_pass_lockstep": (i32, [P, i32, i32, P, P, P]),
            "tsg_smooth_host_batch": (i32, [P, i32, P, C.POINTER(SmoothCfg), P, P, P]),
            "tsg_hilbert_order": (i32, [i64, P, P]),
            "tsg_selftest_alpha": (i32, [P, i64, C.c_uint64, i32, P, P]),
            "tsg_selftest_alpha_cycle": (i32, [P, i64, C.c_uint64, P, P]),
            "tsg_debug_trace": (i32, [P, i64]),
            "tsg_pass": (i32, [P, C.POINTER(SmoothCfg), P, P]),
            "tsg_halo_plan": (i32, [P, P, i64, P, i64]),
            "tsg_halo_pack": (i32, [P, C.c_void_p, i32]),
            "tsg_halo_unpack": (i32, [P, C.c_void_p, i32]),
            "tsg_dist_begin": (i32, [P, C.POINTER(SmoothCfg)]),
            "tsg_mesh_formb_schedule": (i32, [P, i32]),
            "tsg_mesh_side_schedule": (i32, [P, i32]),
            "tsg_dist_pass": (i32, [P, C.POINTER(SmoothCfg), C.c_void_p]),
            "tsg_dist_halo_pack": (i32, [P, C.POINTER(SmoothCfg), C.c_void_p]),
            "tsg_dist_halo_unpack": (i32, [P, C.c_void_p]),
            "tsg_dist_finalize": (i32, [P, C.POINTER(SmoothCfg), C.c_void_p, i32]),
            "tsg_dist_status": (i32, [P, P, P, P]),
            "tsg_dist_end": (i32, [P, C.POINTER(SmoothCfg), P, P, i32, P, P, P]),
            "tsg_quality_tri_alpha": (i32, [P, i64, P, i64, P, P, C.POINTER(QualityReport)]),
            "tsg_quality_vertex_minima": (i32, [P, i64, P, P, i64, P, P]),
            "tsg_peer_local": (i32, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(i64)]),
            "tsg_mesh_slots": (i32, [P, P, i64, P]),
            "tsg_peer_setup": (i32, [P, i32, i32, P, P, P, P, i64, P, P, P]),
            "tsg_peer_prepare": (i32, [P, C.POINTER(SmoothCfg)]),
            "tsg_peer_clear": (i32, [P]),
            "tsg_ipc_handle": (i32, [P, P]),
            "tsg_ipc_open": (i32, [P, P, C.POINTER(P)]),
            "tsg_ipc_close": (i32, [P, P]),
            "tsg_topology": (i32, [P, i64, i64, P, P, P, i64, P, P, P, C.POINTER(i64)]),
            "tsg_debug_layout_check": (i32, [P, C.POINTER(MeshDesc), C.c_char_p, i32]),
            "tsg_hilbert_order_device": (i32, [P, i64, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def check(status: int, what: str):
    if status != TSG_OK:
        raise RuntimeError(f"{what}: {lib().tsg_last_error().decode()} (status {status})")


def hilbert_order(xy: np.ndarray) -> np.ndarray:
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    out = np.empty(len(xy), dtype=np.int64)
    check(lib().tsg_hilbert_order(len(xy), _ptr(xy), _ptr(out)), "tsg_hilbert_order")
    return out


def ipc_handle(dev_ptr: int) -> bytes:
    """CUDA IPC handle (64 bytes) of a device allocation's base pointer (tsg_ipc_handle)."""
    buf = C.create_string_buffer(IPC_HANDLE_BYTES)
    check(lib().tsg_ipc_handle(C.c_void_p(dev_ptr), buf), "tsg_ipc_handle")
    return buf.raw


class Context:
    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        check(lib().tsg_context_create(device, C.byref(self.h)), "tsg_context_create")

    @property
    def stream(self) -> int:
        return lib().tsg_context_stream(self.h) or 0

    def selftest_alpha(self, n=1 << 22, seed=1, newton_steps=1):
        err, bad = C.c_double(), C.c_int64()
        check(lib().tsg_selftest_alpha(self.h, n, seed, newton_steps, C.byref(err), C.byref(bad)),
              "tsg_selftest_alpha")
        return err.value, bad.value

    def selftest_alpha_cycle(self, n=1 << 22, seed=1):
        err, bad = C.c_double(), C.c_int64()
        check(lib().tsg_selftest_alpha_cycle(self.h, n, seed, C.byref(err), C.byref(bad)),
              "tsg_selftest_alpha_cycle")
        return err.value, bad.value

    def quality_tri_alpha(self, xy, tri):
        """Device quality audit of a bare (xy, tri) pair: (alpha per triangle, report dict)."""
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        alpha = np.empty(len(tri))
        rep = QualityReport()
        check(lib().tsg_quality_tri_alpha(self.h, len(xy), _ptr(xy), len(tri), _ptr(tri), _ptr(alpha),
                                          C.byref(rep)), "tsg_quality_tri_alpha")
        return alpha, dict(min_alpha=rep.min_alpha, max_alpha=rep.max_alpha, non_positive=rep.non_positive,
                           histogram=list(rep.histogram))

    def quality_vertex_minima(self, inc_off, inc, alpha):
        inc_off = np.ascontiguousarray(inc_off, dtype=np.int64)
        inc = np.ascontiguousarray(inc, dtype=np.int32)
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        out = np.empty(len(inc_off) - 1)
        check(lib().tsg_quality_vertex_minima(self.h, len(out), _ptr(inc_off), _ptr(inc), len(alpha), _ptr(alpha),
                                              _ptr(out)), "tsg_quality_vertex_minima")
        return out

    def ipc_open(self, handle: bytes) -> int:
        """Maps a peer process's allocation (tsg_ipc_open); returns the device pointer."""
        out = C.c_void_p()
        buf = C.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
        check(lib().tsg_ipc_open(self.h, buf, C.byref(out)), "tsg_ipc_open")
        return out.value

    def ipc_close(self, dev_ptr: int):
        check(lib().tsg_ipc_close(self.h, C.c_void_p(dev_ptr)), "tsg_ipc_close")

    def layout_check(self, xy, tri, topo: dict, order=None) -> str:
        """Builds the device layout on the GPU and on the host; returns the name of the first
        array that differs ("" when identical) — tsg_debug_layout_check."""
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        keep = dict(nbr_off=np.ascontiguousarray(topo["nbr_off"], dtype=np.int64),
                    nbr=np.ascontiguousarray(topo["nbr"], dtype=np.int32),
                    inc_off=np.ascontiguousarray(topo["inc_off"], dtype=np.int64),
                    inc=np.ascontiguousarray(topo["inc"], dtype=np.int32),
                    boundary=np.ascontiguousarray(topo["boundary"], dtype=np.uint8))
        order = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
        d = MeshDesc(len(xy), len(tri), _ptr(xy), _ptr(tri), _ptr(keep["nbr_off"]), _ptr(keep["nbr"]),
                     _ptr(keep["inc_off"]), _ptr(keep["inc"]), _ptr(keep["boundary"]), _ptr(order), 0, 0)
        buf = C.create_string_buffer(64)
        check(lib().tsg_debug_layout_check(self.h, C.byref(d), buf, 64), "tsg_debug_layout_check")
        return buf.value.decode()

    def hilbert_order(self, xy) -> np.ndarray:
        """capi.hilbert_order computed on the device (tsg_hilbert_order_device): same order."""
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        out = np.empty(len(xy), dtype=np.int64)
        check(lib().tsg_hilbert_order_device(self.h, len(xy), _ptr(xy), _ptr(out)), "tsg_hilbert_order_device")
        return out

    def topology(self, nv: int, tri) -> dict:
        """Adjacency + constraints on the device (tsg_topology): same dict as
        paper_1502_00355_b200.topology (find_neighbors / determine_constraints)."""
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        nt = len(tri)
        nbr_off = np.empty(nv + 1, dtype=np.int64)
        inc_off = np.empty(nv + 1, dtype=np.int64)
        nbr = np.empty(max(1, 6 * nt), dtype=np.int32)
        inc = np.empty(max(1, 3 * nt), dtype=np.int32)
        bnd = np.empty(nv, dtype=np.uint8)
        n = C.c_int64()
        check(lib().tsg_topology(self.h, nv, nt, _ptr(tri), _ptr(nbr_off), _ptr(nbr), len(nbr), _ptr(inc_off),
                                 _ptr(inc), _ptr(bnd), C.byref(n)), "tsg_topology")
        # (views: the untouched tail of the 6*nt buffer was never paged in)
        return dict(nbr_off=nbr_off, nbr=nbr[: n.value], inc_off=inc_off, inc=inc[: 3 * nt], boundary=bnd)

    def close(self):
        if self.h:
            lib().tsg_context_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_cfg(form="a", strategy="fused", chunks=1, swap="pingpong", max_iters=100, driver="graph",
             move_tol=0.0, bbox_diag=0.0) -> SmoothCfg:
    return SmoothCfg(FORM[form], STRATEGY[strategy], chunks, SWAP[swap], max_iters, DRIVER[driver],
                     move_tol, bbox_diag)


class DeviceMesh:
    """A tsg_mesh: upload from host arrays (original numbering)."""

    def __init__(self, ctx: Context, xy, tri, topo, layout="aos", precision="f64", order=None):
        """topo: the host adjacency dict (tsg_mesh_upload), or None to build it on the device
        inside the upload (tsg_mesh_upload_triangles: no host round trip of the adjacency)."""
        self.ctx = ctx
        self.xy = np.ascontiguousarray(xy, dtype=np.float64)
        self.tri = np.ascontiguousarray(tri, dtype=np.int32)
        self.nv, self.nt = len(self.xy), len(self.tri)
        if topo is None:
            order = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
            d = MeshDesc(self.nv, self.nt, _ptr(self.xy), _ptr(self.tri), None, None, None, None, None, _ptr(order),
                         LAYOUT[layout], PRECISION[precision])
            self.h = C.c_void_p()
            check(lib().tsg_mesh_upload_triangles(ctx.h, C.byref(d), C.byref(self.h)), "tsg_mesh_upload_triangles")
            return
        keep = dict(nbr_off=np.ascontiguousarray(topo["nbr_off"], dtype=np.int64),
                    nbr=np.ascontiguousarray(topo["nbr"], dtype=np.int32),
                    inc_off=np.ascontiguousarray(topo["inc_off"], dtype=np.int64),
                    inc=np.ascontiguousarray(topo["inc"], dtype=np.int32),
                    boundary=np.ascontiguousarray(topo["boundary"], dtype=np.uint8))
        order = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
        d = MeshDesc(self.nv, self.nt, _ptr(self.xy), _ptr(self.tri), _ptr(keep["nbr_off"]),
                     _ptr(keep["nbr"]), _ptr(keep["inc_off"]), _ptr(keep["inc"]),
                     _ptr(keep["boundary"]), _ptr(order), LAYOUT[layout], PRECISION[precision])
        self.h = C.c_void_p()
        check(lib().tsg_mesh_upload(ctx.h, C.byref(d), C.byref(self.h)), "tsg_mesh_upload")

    def free(self):
        if self.h:
            lib().tsg_mesh_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        return int(lib().tsg_mesh_device_bytes(self.h))

    def set_coords(self, xy):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        check(lib().tsg_mesh_set_coords(self.h, _ptr(xy)), "tsg_mesh_set_coords")

    def restore_coords(self):
        check(lib().tsg_mesh_restore_coords(self.h), "tsg_mesh_restore_coords")

    def get_coords(self) -> np.ndarray:
        out = np.empty((self.nv, 2))
        check(lib().tsg_mesh_get_coords(self.h, _ptr(out)), "tsg_mesh_get_coords")
        return out

    def tri_alpha(self) -> np.ndarray:
        out = np.empty(self.nt)
        check(lib().tsg_tri_alpha(self.h, _ptr(out)), "tsg_tri_alpha")
        return out

    def vertex_minima(self) -> np.ndarray:
        out = np.empty(self.nv)
        check(lib().tsg_vertex_minima(self.h, _ptr(out)), "tsg_vertex_minima")
        return out

    def alpha_extrema(self):
        lo, hi, n = C.c_double(), C.c_double(), C.c_int64()
        check(lib().tsg_alpha_extrema(self.h, C.byref(lo), C.byref(hi), C.byref(n)), "tsg_alpha_extrema")
        return lo.value, hi.value, n.value

    def smooth(self, cfg: SmoothCfg):
        st = SmoothStats()
        acc = np.zeros(cfg.max_iters, dtype=np.int32)
        md = np.zeros(cfg.max_iters)
        check(lib().tsg_smooth(self.h, C.byref(cfg), C.byref(st), _ptr(acc), _ptr(md), cfg.max_iters),
              "tsg_smooth")
        it = st.iterations
        return dict(iterations=it, stop=STOP[st.stop], accepted=acc[:it], max_disp=md[:it],
                    device_ms=st.device_ms, node_kernel_ms=st.node_kernel_ms, launches=st.launches,
                    schedule=SCHEDULE.get(st.schedule, str(st.schedule)),
                    node_updates=st.node_updates)

    def smooth_host(self, xy_in, cfg: SmoothCfg, xy_out=None):
        xy_in = np.ascontiguousarray(xy_in, dtype=np.float64)
        if xy_out is None:
            xy_out = np.empty_like(xy_in)
        st = SmoothStats()
        acc = np.zeros(cfg.max_iters, dtype=np.int32)
        md = np.zeros(cfg.max_iters)
        check(lib().tsg_smooth_host(self.h, _ptr(xy_in), C.byref(cfg), _ptr(xy_out), C.byref(st),
                                    _ptr(acc), _ptr(md), cfg.max_iters), "tsg_smooth_host")
        it = st.iterations
        return xy_out, dict(iterations=it, stop=STOP[st.stop], accepted=acc[:it], max_disp=md[:it],
                            device_ms=st.device_ms, launches=st.launches)

    def smooth_host_batch(self, xy_ins, cfg: SmoothCfg, xy_outs):
        """tsg_smooth_host_batch: smooths every coordinate set of `xy_ins` (host arrays, ideally
        pinned) into the matching array of `xy_outs`, copies overlapped with the passes.
        Returns (iterations, stop names) per item."""
        n = len(xy_ins)
        assert len(xy_outs) == n
        for a in list(xy_ins) + list(xy_outs):
            assert a.dtype == np.float64 and a.flags.c_contiguous and a.shape == (self.nv, 2)
        ins = (C.c_void_p * max(1, n))(*[a.ctypes.data for a in xy_ins])
        outs = (C.c_void_p * max(1, n))(*[a.ctypes.data for a in xy_outs])
        it = np.zeros(max(1, n), dtype=np.int32)
        stop = np.zeros(max(1, n), dtype=np.int32)
        check(lib().tsg_smooth_host_batch(self.h, n, ins, C.byref(cfg), outs, _ptr(it), _ptr(stop)),
              "tsg_smooth_host_batch")
        return it[:n].copy(), [STOP[x] for x in stop[:n]]

    def pass_lockstep(self, form="a", chunks=1):
        dec = np.empty(self.nv, dtype=np.int8)
        acc = C.c_int32()
        md = C.c_double()
        check(lib().tsg_pass_lockstep(self.h, FORM[form], chunks, _ptr(dec), C.byref(acc), C.byref(md)),
              "tsg_pass_lockstep")
        return dec, acc.value, md.value

    # ---- multi-GPU partitions ----
    def run_pass(self, cfg: SmoothCfg):
        acc, md = C.c_int32(), C.c_double()
        check(lib().tsg_pass(self.h, C.byref(cfg), C.byref(acc), C.byref(md)), "tsg_pass")
        return acc.value, md.value

    def halo_plan(self, send_ids, recv_ids):
        self._send = np.ascontiguousarray(send_ids, dtype=np.int64)
        self._recv = np.ascontiguousarray(recv_ids, dtype=np.int64)
        check(lib().tsg_halo_plan(self.h, _ptr(self._send), len(self._send), _ptr(self._recv), len(self._recv)),
              "tsg_halo_plan")

    def halo_pack(self, out_ptr: int, on_host: bool):
        """Writes 2*n_send doubles at out_ptr (device pointer, or host pointer if on_host)."""
        check(lib().tsg_halo_pack(self.h, C.c_void_p(out_ptr), 1 if on_host else 0), "tsg_halo_pack")

    def halo_unpack(self, in_ptr: int, on_host: bool):
        check(lib().tsg_halo_unpack(self.h, C.c_void_p(in_ptr), 1 if on_host else 0), "tsg_halo_unpack")

    def formb_schedule(self, mode: str):
        """Form B schedule: "auto", "levels" (a launch per dependency level) or "chunks" (one CTA
        per chunk walking its levels).  Results are identical."""
        check(lib().tsg_mesh_formb_schedule(self.h, {"auto": 0, "levels": 1, "chunks": 2, "flow": 3}[mode]),
              "tsg_mesh_formb_schedule")

    def side_schedule(self, mode: str):
        """Form A fused rows of valence >= 32: "auto", "kernels" (per-tier grids after the tile
        grid) or "persist" (a persistent kernel beside it).  Results are identical."""
        check(lib().tsg_mesh_side_schedule(self.h, {"auto": 0, "kernels": 1, "persist": 2}[mode]),
              "tsg_mesh_side_schedule")

    # ---- peer-memory partitioned driver (include/tsg.h, tsg_peer_*) ----
    def peer_local(self):
        """(buf0, buf1, sync, nv): this mesh's coordinate buffers and sync block (device ptrs)."""
        b0, b1, sy, nv = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_int64()
        check(lib().tsg_peer_local(self.h, C.byref(b0), C.byref(b1), C.byref(sy), C.byref(nv)), "tsg_peer_local")
        return b0.value, b1.value, sy.value, nv.value

    def slots(self, ids) -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.empty(len(ids), dtype=np.int64)
        check(lib().tsg_mesh_slots(self.h, _ptr(ids), len(ids), _ptr(out)), "tsg_mesh_slots")
        return out

    def peer_setup(self, rank, world, buf0s, buf1s, syncs, nvs, push_peer, push_src, push_dst):
        arr = lambda xs: (C.c_void_p * len(xs))(*xs)
        nvs = np.ascontiguousarray(nvs, dtype=np.int64)
        self._push = (np.ascontiguousarray(push_peer, dtype=np.int32), np.ascontiguousarray(push_src, dtype=np.int64),
                      np.ascontiguousarray(push_dst, dtype=np.int64))
        check(lib().tsg_peer_setup(self.h, rank, world, arr(buf0s), arr(buf1s), arr(syncs), _ptr(nvs),
                                   len(self._push[0]), _ptr(self._push[0]), _ptr(self._push[1]), _ptr(self._push[2])),
              "tsg_peer_setup")

    def peer_prepare(self, cfg: SmoothCfg):
        check(lib().tsg_peer_prepare(self.h, C.byref(cfg)), "tsg_peer_prepare")

    def peer_clear(self):
        check(lib().tsg_peer_clear(self.h), "tsg_peer_clear")

    # Device-resident partitioned loop (include/tsg.h, tsg_dist_*): enqueue-only calls taking
    # device pointers (e.g. torch CUDA tensors' data_ptr()).
    def dist_begin(self, cfg: SmoothCfg):
        check(lib().tsg_dist_begin(self.h, C.byref(cfg)), "tsg_dist_begin")

    def dist_pass(self, cfg: SmoothCfg, stats_ptr: int):
        check(lib().tsg_dist_pass(self.h, C.byref(cfg), C.c_void_p(stats_ptr)), "tsg_dist_pass")

    def dist_halo_pack(self, cfg: SmoothCfg, out_ptr: int):
        check(lib().tsg_dist_halo_pack(self.h, C.byref(cfg), C.c_void_p(out_ptr)), "tsg_dist_halo_pack")

    def dist_halo_unpack(self, in_ptr: int):
        check(lib().tsg_dist_halo_unpack(self.h, C.c_void_p(in_ptr)), "tsg_dist_halo_unpack")

    def dist_finalize(self, cfg: SmoothCfg, gathered_ptr: int, n_parts: int):
        check(lib().tsg_dist_finalize(self.h, C.byref(cfg), C.c_void_p(gathered_ptr), n_parts), "tsg_dist_finalize")

    def dist_status(self):
        it, done, stop = C.c_int32(), C.c_int32(), C.c_int32()
        check(lib().tsg_dist_status(self.h, C.byref(it), C.byref(done), C.byref(stop)), "tsg_dist_status")
        return it.value, bool(done.value), STOP[stop.value]

    def dist_end(self, cfg: SmoothCfg):
        cap = max(1, cfg.max_iters)
        acc = np.zeros(cap, dtype=np.int32)
        md = np.zeros(cap, dtype=np.float64)
        it, stop, launches = C.c_int32(), C.c_int32(), C.c_int64()
        check(lib().tsg_dist_end(self.h, C.byref(cfg), _ptr(acc), _ptr(md), cap, C.byref(it), C.byref(stop),
                                 C.byref(launches)), "tsg_dist_end")
        n = it.value
        self.dist_launches = launches.value
        return n, STOP[stop.value], acc[:n].copy(), md[:n].copy()
