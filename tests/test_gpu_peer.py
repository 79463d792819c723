"""Partitioned Form A over peer memory (csrc/tsg_peer.cuh, tsg_peer_*): W partitions of one
mesh, each a device mesh with its own context and stream on cuda:0, wired to each other with
raw device pointers (distributed.connect_peers_local) exactly as separate GPUs are over CUDA
IPC; each partition's smooth() (one graph per rank: node kernels, direct halo stores into the
peers' buffers, flag barrier with the global stop statistics) runs from its own host thread.
The gathered owned coordinates, per-pass statistics and stop must equal one mesh's run bit for
bit (Form A on N GPUs == 1 GPU), across repeated runs (monotonic barrier ticks)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_all(meshes, cfg):
    out = [None] * len(meshes)
    err = []

    def go(r):
        try:
            out[r] = meshes[r].smooth(cfg)
        except Exception as exc:  # reported below
            err.append(exc)

    th = [threading.Thread(target=go, args=(r,)) for r in range(len(meshes))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not err, err
    return out


@pytest.mark.parametrize("world,kind,tol", [(2, "delaunay", 0.0), (3, "graded", 1e-6), (4, "grid", 1e-6)])
def test_peer_partitions_equal_one_mesh(capi, ts, world, kind, tol):
    from paper_1502_00355_b200 import distributed as D

    if kind == "delaunay":
        xy, tri = ts.delaunay_arrays(30000, 8)
    elif kind == "graded":
        xy, tri = ts.graded_arrays(30000, 2, 3e-3, 300)
    else:
        xy, tri = ts.grid_arrays(150, 170, 0.3, 4)
    topo = ts.topology(len(xy), tri)
    diag = ts.bbox_diagonal(xy)
    cfg = capi.make_cfg(form="a", max_iters=40, move_tol=tol, bbox_diag=diag)
    ctx0 = capi.Context(0)
    ref = capi.DeviceMesh(ctx0, xy, tri, topo, order=capi.hilbert_order(xy))
    want = ref.smooth(cfg)
    want_xy = ref.get_coords()
    ref.free()

    owner = D.owners_by_weight(capi.hilbert_order(xy), 1 + np.diff(topo["nbr_off"]), world)
    parts = [D.build_partition(r, world, owner, xy, tri, topo) for r in range(world)]
    ctxs = [capi.Context(0) for _ in parts]
    meshes = [capi.DeviceMesh(c, p.xy, p.tri, p.topo, order=capi.hilbert_order(p.xy)) for c, p in zip(ctxs, parts)]
    D.connect_peers_local(meshes, parts)
    for m in meshes:  # allocations / capture before any rank's barrier spins on the shared device
        m.peer_prepare(cfg)
    for rep in range(2):
        for m, p in zip(meshes, parts):
            m.set_coords(p.xy)
        res = _run_all(meshes, cfg)
        full = np.full_like(xy, np.nan)
        for m, p, r in zip(meshes, parts, res):
            assert r["iterations"] == want["iterations"] and r["stop"] == want["stop"], (rep, r["iterations"])
            assert np.array_equal(r["accepted"], want["accepted"])
            assert np.array_equal(r["max_disp"].view(np.uint64), want["max_disp"].view(np.uint64))
            full[p.gids[p.owned]] = m.get_coords()[p.owned]
        assert np.array_equal(full.view(np.uint64), want_xy.view(np.uint64)), rep
    # back to a single-mesh run on a partition (halo pinned): the peer graph is dropped
    meshes[0].peer_clear()
    meshes[0].set_coords(parts[0].xy)
    meshes[0].smooth(capi.make_cfg(form="a", max_iters=3))
    for m in meshes:
        m.free()


def _ipc_worker(rank, world, port_num, part_dir, passes, out_path):
    import os
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from paper_1502_00355_b200 import capi, distributed as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_num}", rank=rank, world_size=world)
    part, meta = D.load_partition(part_dir, rank)
    ctx = capi.Context(0)
    mesh = capi.DeviceMesh(ctx, part.xy, part.tri, part.topo, order=capi.hilbert_order(part.xy))
    opened = D.connect_peers_ipc(ctx, mesh, part, dist)
    cfg = capi.make_cfg(form="a", max_iters=passes, move_tol=0.0, bbox_diag=meta["bbox_diag"])
    mesh.peer_prepare(cfg)
    dist.barrier()
    r = mesh.smooth(cfg)
    full = D.gather_coords(part, mesh.get_coords()[part.owned], meta["nv"])
    if rank == 0:
        np.savez(out_path, xy=full, acc=r["accepted"], it=r["iterations"])
    dist.barrier()
    for p in opened:
        ctx.ipc_close(p)
    mesh.free()
    ctx.close()
    dist.destroy_process_group()


def test_peer_partitions_over_cuda_ipc_processes(capi, ts, tmp_path):
    """One process per partition (two processes sharing cuda:0), buffers shared as CUDA IPC
    handles (distributed.connect_peers_ipc, the bench's --transport p2p): the gathered result
    equals one mesh's run bit for bit."""
    import socket

    import torch.multiprocessing as mp

    from paper_1502_00355_b200 import distributed as D

    xy, tri = ts.delaunay_arrays(20000, 12)
    topo = ts.topology(len(xy), tri)
    world, passes = 2, 8
    owner = D.owners_by_order(capi.hilbert_order(xy), world)
    part_dir = str(tmp_path / "parts")
    D.write_partitions(part_dir, world, owner, xy, tri, topo, ts.bbox_diagonal(xy))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_num = s.getsockname()[1]
    out = str(tmp_path / "r.npz")
    mp.spawn(_ipc_worker, args=(world, port_num, part_dir, passes, out), nprocs=world, join=True)
    r = np.load(out)
    ctx = capi.Context(0)
    ref = capi.DeviceMesh(ctx, xy, tri, topo)
    want = ref.smooth(capi.make_cfg(form="a", max_iters=passes, move_tol=0.0))
    assert int(r["it"]) == want["iterations"] and np.array_equal(r["acc"], want["accepted"])
    assert np.array_equal(r["xy"].view(np.uint64), ref.get_coords().view(np.uint64))
    ref.free()
