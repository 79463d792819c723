"""Multi-GPU Smart Laplacian: one process per GPU, the vertex set partitioned.

Partitioning: contiguous ranges of a locality order (Hilbert curve over the coordinates) —
near-optimal cuts on planar meshes, O(n log n).  Rank r *owns* the vertices of its range; its
device mesh holds the owned vertices plus a one-ring **halo** (every vertex of a triangle that
touches an owned vertex), numbered locally in ascending global id so that neighbour sums keep
the reference's ascending-id order.  Halo vertices are pinned locally.

Two drivers: `smooth_partitioned` (host-synchronous per pass: simple, used by the CPU-side
tests) and `DeviceLoop` (device-resident: the pass, the halo exchange, the stats all-gather and the
stop rule are all enqueued on the engine's stream, NCCL ordered on it, the host polls every 8
passes — the multi-GPU bench path).

One pass (Form A, Jacobi — every read is pass-start) =
  1. `tsg_pass` on every rank (owned movable vertices updated on the device);
  2. halo exchange: each rank packs the new coordinates of its vertices that lie in other
     ranks' halos (`tsg_halo_pack`), an all-to-all moves them (NCCL over NVLink with device
     buffers, or gloo with host buffers), `tsg_halo_unpack` writes them into the halo slots;
  3. all-reduce of {accepted (sum), max displacement (max)} and the reference's stop rule
     (`src/smoothing.cpp:132-141`), identical on every rank.
Because every owned update reads exactly the pass-start values the single-GPU pass reads, the
result is bit-identical to one GPU (tests/test_distributed.py, tests/test_gpu_distributed.py).

Form B is partition-dependent (chunks are original-id ranges, in-chunk reads are live), so the
partitioned driver supports Form A; Form B with chunk-aligned partitions is DESIGN.md §9 "next".
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

STOP_NAMES = ("max_iters", "displacement", "no_moves")


def owners_by_order(order: np.ndarray, world: int) -> np.ndarray:
    """owner[v] for contiguous, equally sized ranges of the locality order."""
    nv = len(order)
    owner = np.empty(nv, dtype=np.int32)
    owner[order] = (np.arange(nv, dtype=np.int64) * world // nv).astype(np.int32)
    return owner


def owners_by_weight(order: np.ndarray, weight: np.ndarray, world: int) -> np.ndarray:
    """owner[v] for contiguous ranges of the locality order holding equal total `weight`
    (e.g. 1 + valence: a rank's pass time grows with its rows' lengths, so graded meshes with
    hubs are cut by work, not by vertex count)."""
    nv = len(order)
    w = np.asarray(weight, dtype=np.float64)[order]
    cum = np.cumsum(w)
    total = cum[-1] if nv else 0.0
    # vertex at position i goes to rank floor(world * (cum[i] - w[i] / 2) / total)
    mid = cum - 0.5 * w
    rank_of_pos = np.minimum((mid * world / max(total, 1e-300)).astype(np.int64), world - 1)
    owner = np.empty(nv, dtype=np.int32)
    owner[order] = rank_of_pos.astype(np.int32)
    return owner


def _gather_rows(off: np.ndarray, vals: np.ndarray, rows: np.ndarray):
    """CSR rows `rows` of (off, vals) -> (new_off int64, new_vals)."""
    lens = off[rows + 1] - off[rows]
    new_off = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=new_off[1:])
    total = int(new_off[-1])
    if total == 0:
        return new_off, vals[:0].copy()
    starts = np.repeat(off[rows] - new_off[:-1], lens)
    idx = starts + np.arange(total, dtype=np.int64)
    return new_off, vals[idx]


@dataclass
class Partition:
    rank: int
    world: int
    gids: np.ndarray            # local id -> global id (ascending)
    owned: np.ndarray           # bool per local vertex
    xy: np.ndarray              # (n_local, 2)
    tri: np.ndarray             # (nt_local, 3) local ids
    topo: dict                  # local topology (halo rows empty and pinned)
    send_ids: np.ndarray        # local ids, grouped by peer rank, ascending global id within
    send_counts: list = field(default_factory=list)
    recv_ids: np.ndarray = None  # local halo ids, same grouping
    recv_counts: list = field(default_factory=list)

    @property
    def n_owned(self) -> int:
        return int(self.owned.sum())


def build_partition(rank: int, world: int, owner: np.ndarray, xy: np.ndarray, tri: np.ndarray,
                    topo: dict) -> Partition:
    nv = len(xy)
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    own_g = owner == rank
    tmask = own_g[tri].any(axis=1)
    tri_g = tri[tmask]
    local = np.union1d(np.nonzero(own_g)[0], np.unique(tri_g))  # ascending global ids
    n = len(local)
    g2l = np.full(nv, -1, dtype=np.int64)
    g2l[local] = np.arange(n)
    tri_l = g2l[tri_g].astype(np.int32)
    tri_g2l = np.full(len(tri), -1, dtype=np.int64)
    tri_g2l[np.nonzero(tmask)[0]] = np.arange(len(tri_g))
    owned_l = own_g[local]

    # Owned rows come from the global topology (complete: every incident triangle and neighbour
    # of an owned vertex is local); halo rows are empty and the halo is pinned.
    rows = local
    nbr_off, nbr = _gather_rows(np.asarray(topo["nbr_off"]), np.asarray(topo["nbr"]), rows)
    inc_off, inc = _gather_rows(np.asarray(topo["inc_off"]), np.asarray(topo["inc"]), rows)
    keep_n = np.repeat(owned_l, np.diff(nbr_off))
    keep_i = np.repeat(owned_l, np.diff(inc_off))
    nbr_off2 = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.where(owned_l, np.diff(nbr_off), 0), out=nbr_off2[1:])
    inc_off2 = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.where(owned_l, np.diff(inc_off), 0), out=inc_off2[1:])
    topo_l = {
        "nbr_off": nbr_off2,
        "nbr": g2l[nbr[keep_n]].astype(np.int32),
        "inc_off": inc_off2,
        "inc": tri_g2l[inc[keep_i]].astype(np.int32),
        "boundary": np.where(owned_l, np.asarray(topo["boundary"])[local], 1).astype(np.uint8),
    }
    assert (topo_l["nbr"] >= 0).all() and (topo_l["inc"] >= 0).all()

    # Send sets: my vertices that share a triangle with a vertex owned by peer q.
    corner_owner = owner[tri]
    send = [[] for _ in range(world)]
    for a in range(3):
        for b in range(3):
            if a == b:
                continue
            m = (corner_owner[:, a] == rank) & (corner_owner[:, b] != rank)
            if m.any():
                for q in np.unique(corner_owner[m, b]):
                    send[int(q)].append(tri[m & (corner_owner[:, b] == q), a])
    send_ids, send_counts = [], []
    for q in range(world):
        g = np.unique(np.concatenate(send[q])) if send[q] else np.zeros(0, dtype=np.int64)
        send_ids.append(g2l[g])
        send_counts.append(len(g))
    halo_g = local[~owned_l]
    recv_ids, recv_counts = [], []
    for q in range(world):
        g = halo_g[owner[halo_g] == q]  # ascending global id
        recv_ids.append(g2l[g])
        recv_counts.append(len(g))
    return Partition(rank, world, local, owned_l, np.ascontiguousarray(xy[local]), tri_l, topo_l,
                     np.concatenate(send_ids).astype(np.int64), send_counts,
                     np.concatenate(recv_ids).astype(np.int64), recv_counts)


# ---- per-rank partition files: the mesh is prepared once, every rank loads only its part ----

_PART_FIELDS = ("gids", "owned", "xy", "tri", "send_ids", "recv_ids")
_TOPO_FIELDS = ("nbr_off", "nbr", "inc_off", "inc", "boundary")


def write_partitions(out_dir: str, world: int, owner: np.ndarray, xy: np.ndarray, tri: np.ndarray, topo: dict,
                     bbox_diag: float) -> list:
    """Builds every rank's Partition from the global mesh (once, on one host process) and
    writes `part_<r>.npz` per rank plus `meta.npz` (nv, nt, world, bbox diagonal) into
    `out_dir`.  A rank then needs only its own file (`load_partition`): no rank holds the
    global mesh or builds the global topology.  Returns the file paths."""
    import os

    os.makedirs(out_dir, exist_ok=True)
    paths = []
    for r in range(world):
        p = build_partition(r, world, owner, xy, tri, topo)
        arrays = {k: getattr(p, k) for k in _PART_FIELDS}
        arrays.update({"topo_" + k: np.asarray(p.topo[k]) for k in _TOPO_FIELDS})
        arrays["send_counts"] = np.asarray(p.send_counts, dtype=np.int64)
        arrays["recv_counts"] = np.asarray(p.recv_counts, dtype=np.int64)
        path = os.path.join(out_dir, f"part_{r}.npz")
        np.savez(path, **arrays)
        paths.append(path)
    np.savez(os.path.join(out_dir, "meta.npz"), nv=len(xy), nt=len(tri), world=world, bbox_diag=bbox_diag)
    return paths


def load_partition(out_dir: str, rank: int):
    """(Partition, meta dict) of `rank` from write_partitions' files."""
    import os

    meta = dict(np.load(os.path.join(out_dir, "meta.npz")))
    world = int(meta["world"])
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside the partition set of {world}")
    z = np.load(os.path.join(out_dir, f"part_{rank}.npz"))
    topo = {k: z["topo_" + k] for k in _TOPO_FIELDS}
    part = Partition(rank, world, z["gids"], z["owned"], z["xy"], z["tri"], topo, z["send_ids"],
                     [int(c) for c in z["send_counts"]], z["recv_ids"], [int(c) for c in z["recv_counts"]])
    return part, {k: (float(v) if k == "bbox_diag" else int(v)) for k, v in meta.items()}


class DeviceEngine:
    """A partition on one GPU through the C ABI (paper_1502_00355_b200.capi)."""

    def __init__(self, ctx, part: Partition, layout="aos", precision="f64", reorder=True):
        from . import capi

        self.capi = capi
        order = capi.hilbert_order(part.xy) if reorder else None
        self.mesh = capi.DeviceMesh(ctx, part.xy, part.tri, part.topo, layout=layout, precision=precision,
                                    order=order)
        self.mesh.halo_plan(part.send_ids, part.recv_ids)
        self.part = part

    def run_pass(self, cfg):
        _require_form_a(cfg)
        return self.mesh.run_pass(cfg)

    def pack(self, buf):
        """Writes the send vertices' coordinates into `buf` (torch float64, device or host)."""
        self.mesh.halo_pack(buf.data_ptr(), not buf.is_cuda)

    def unpack(self, buf):
        self.mesh.halo_unpack(buf.data_ptr(), not buf.is_cuda)

    def owned_coords(self) -> np.ndarray:
        return self.mesh.get_coords()[self.part.owned]


class Exchanger:
    """All-to-all of halo coordinates + the stats all-reduce over torch.distributed.

    device=True: CUDA tensors (NCCL over NVLink); the engine packs straight into them.
    device=False: host tensors (gloo)."""

    def __init__(self, part: Partition, device: bool, torch_device=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.part = part
        self.device = device
        dev = torch_device if device else torch.device("cpu")
        self.send = torch.empty(2 * max(1, len(part.send_ids)), dtype=torch.float64, device=dev)
        self.recv = torch.empty(2 * max(1, len(part.recv_ids)), dtype=torch.float64, device=dev)
        self.stat_sum = torch.zeros(1, dtype=torch.int64, device=dev)
        self.stat_max = torch.zeros(1, dtype=torch.float64, device=dev)
        self.in_splits = [2 * c for c in part.send_counts]
        self.out_splits = [2 * c for c in part.recv_counts]

    def exchange(self, engine):
        n_s, n_r = len(self.part.send_ids), len(self.part.recv_ids)
        if n_s:
            engine.pack(self.send[: 2 * n_s])
        self.dist.all_to_all_single(self.recv[: 2 * n_r], self.send[: 2 * n_s], self.out_splits, self.in_splits)
        if n_r:
            engine.unpack(self.recv[: 2 * n_r])

    def reduce_stats(self, accepted: int, max_disp: float):
        self.stat_sum.fill_(accepted)
        self.stat_max.fill_(max_disp)
        self.dist.all_reduce(self.stat_sum, op=self.dist.ReduceOp.SUM)
        self.dist.all_reduce(self.stat_max, op=self.dist.ReduceOp.MAX)
        return int(self.stat_sum.item()), float(self.stat_max.item())


def _require_form_a(cfg):
    """Partitions are exact for Form A only: a Form B vertex reads in-chunk values written
    earlier in the same pass, so a partition boundary inside a chunk would change results."""
    if cfg is not None and cfg.form != 0:
        raise ValueError("partitioned smoothing supports Form A only (Form B reads live in-chunk "
                         "values; see DESIGN.md §6)")


def smooth_partitioned(engine, exchanger: Exchanger, cfg, max_iters: int, move_tol: float, bbox_diag: float):
    """The reference pass loop (src/smoothing.cpp:98-141) over partitions.  Returns
    (iterations, stop, accepted_per_pass, max_disp_per_pass)."""
    _require_form_a(cfg)
    tol_abs = move_tol * bbox_diag
    accepted, max_disp = [], []
    stop = "max_iters"
    for _ in range(max_iters):
        acc, md = engine.run_pass(cfg)
        exchanger.exchange(engine)
        acc, md = exchanger.reduce_stats(acc, md)
        accepted.append(acc)
        max_disp.append(md)
        if acc == 0:
            stop = "no_moves"
            break
        if md < tol_abs:
            stop = "displacement"
            break
    return len(accepted), stop, accepted, max_disp


class DeviceLoop:
    """The device-resident pass loop (include/tsg.h, tsg_dist_*): per pass the node kernels, the
    halo exchange and the all-gather of {accepted, max displacement} are all ENQUEUED on the
    engine's stream — NCCL collectives are ordered on it through torch's current stream — and the
    stop rule runs on the device; the host polls the stop flag every `check_every` passes.  With
    host (gloo) buffers the exchange and the all-gather go through host copies (testing)."""

    def __init__(self, engine, part: Partition, device: bool, torch_device, stream_ptr: int):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.engine, self.part, self.device = torch, dist, engine, part, device
        self.dev = torch_device
        self.stream = torch.cuda.ExternalStream(stream_ptr, device=torch_device)
        n_s, n_r = len(part.send_ids), len(part.recv_ids)
        self.n_s, self.n_r = n_s, n_r
        self.send = torch.empty(2 * max(1, n_s), dtype=torch.float64, device=torch_device)
        self.recv = torch.empty(2 * max(1, n_r), dtype=torch.float64, device=torch_device)
        self.stats = torch.zeros(2, dtype=torch.float64, device=torch_device)  # {accepted, max disp}
        self.gathered = torch.zeros(2 * part.world, dtype=torch.float64, device=torch_device)
        self.in_splits = [2 * c for c in part.send_counts]
        self.out_splits = [2 * c for c in part.recv_counts]

    def _exchange(self, cfg):
        mesh, dist = self.engine.mesh, self.dist
        if self.n_s:
            mesh.dist_halo_pack(cfg, self.send.data_ptr())
        if self.device:
            dist.all_to_all_single(self.recv[: 2 * self.n_r], self.send[: 2 * self.n_s], self.out_splits,
                                   self.in_splits)
        else:
            recv = self.recv[: 2 * self.n_r].cpu()
            dist.all_to_all_single(recv, self.send[: 2 * self.n_s].cpu(), self.out_splits, self.in_splits)
            self.recv[: 2 * self.n_r].copy_(recv)
        if self.n_r:
            mesh.dist_halo_unpack(self.recv.data_ptr())

    def _gather(self):
        if self.device:
            self.dist.all_gather_into_tensor(self.gathered, self.stats)
        else:
            out = [self.torch.empty(2, dtype=self.torch.float64) for _ in range(self.part.world)]
            self.dist.all_gather(out, self.stats.cpu())
            self.gathered.copy_(self.torch.cat(out))

    def smooth(self, cfg, check_every: int = 8):
        """Runs cfg.max_iters passes at most (stop rule on the global totals).  Returns
        (iterations, stop, accepted_per_pass, max_disp_per_pass)."""
        mesh = self.engine.mesh
        mesh.dist_begin(cfg)
        with self.torch.cuda.stream(self.stream):
            for q in range(cfg.max_iters):
                mesh.dist_pass(cfg, self.stats.data_ptr())
                self._exchange(cfg)
                self._gather()
                mesh.dist_finalize(cfg, self.gathered.data_ptr(), self.part.world)
                if (q + 1) % check_every == 0 and mesh.dist_status()[1]:
                    break
        return mesh.dist_end(cfg)


# ---- peer-memory partitioned loop (tsg_peer_*: halo stores and barrier inside the graph) ----

def _groups(ids: np.ndarray, counts) -> list:
    out, o = [], 0
    for c in counts:
        out.append(ids[o:o + c])
        o += c
    return out


def peer_info(mesh, part: Partition) -> dict:
    """What the other ranks need from this rank: its buffers / sync block, its vertex count, and
    for every sender q the device slots of the halo vertices q sends (in q's send order:
    ascending global id on both sides)."""
    b0, b1, sync, nv = mesh.peer_local()
    recv = _groups(part.recv_ids, part.recv_counts)
    return {"rank": part.rank, "ptrs": (b0, b1, sync), "nv": nv, "recv_slots": [mesh.slots(g) for g in recv]}


def connect_peers(mesh, part: Partition, infos: list, mapped: list):
    """tsg_peer_setup from every rank's peer_info and the peers' pointers as mapped in this
    process (`mapped[r] = (buf0, buf1, sync)`; entry `part.rank` = this mesh's own)."""
    send = _groups(part.send_ids, part.send_counts)
    peer, src, dst = [], [], []
    for r in range(part.world):
        if r == part.rank or len(send[r]) == 0:
            continue
        d = infos[r]["recv_slots"][part.rank]
        if len(d) != len(send[r]):
            raise RuntimeError(f"rank {part.rank} sends {len(send[r])} vertices to {r}, which expects {len(d)}")
        peer.append(np.full(len(d), r, dtype=np.int32))
        src.append(send[r])
        dst.append(d)
    cat = lambda xs, t: np.concatenate(xs).astype(t) if xs else np.zeros(0, dtype=t)
    mesh.peer_setup(part.rank, part.world, [m[0] for m in mapped], [m[1] for m in mapped], [m[2] for m in mapped],
                    [i["nv"] for i in infos], cat(peer, np.int32), cat(src, np.int64), cat(dst, np.int64))


def connect_peers_local(meshes: list, parts: list):
    """All partitions in this process (one device or several): raw device pointers."""
    infos = [peer_info(m, p) for m, p in zip(meshes, parts)]
    for m, p in zip(meshes, parts):
        connect_peers(m, p, infos, [i["ptrs"] for i in infos])


def connect_peers_ipc(ctx, mesh, part: Partition, dist) -> list:
    """One process per GPU: the buffers are shared as CUDA IPC handles through
    torch.distributed (all_gather_object) and mapped with tsg_ipc_open.  Returns the mapped
    pointers to release with ctx.ipc_close after the last smooth."""
    from . import capi

    info = peer_info(mesh, part)
    own = info.pop("ptrs")
    info["handles"] = tuple(capi.ipc_handle(p) for p in own)
    infos = [None] * part.world
    dist.all_gather_object(infos, info)
    mapped, opened = [], []
    for r, inf in enumerate(infos):
        if r == part.rank:
            mapped.append(own)
        else:
            ptrs = tuple(ctx.ipc_open(h) for h in inf["handles"])
            mapped.append(ptrs)
            opened.extend(ptrs)
    connect_peers(mesh, part, infos, mapped)
    return opened


def gather_coords(part: Partition, owned_xy: np.ndarray, nv: int):
    """All owned coordinates to every rank (gloo / nccl object gather), in global order."""
    import torch.distributed as dist

    pieces = [None] * part.world
    dist.all_gather_object(pieces, (part.gids[part.owned], owned_xy))
    out = np.empty((nv, 2))
    for gids, xy in pieces:
        out[gids] = xy
    return out
