"""Multi-process partitioned smoothing on CPU (gloo, world_size 2 and 3): the host-side
partition / halo / all-to-all / stop-rule logic of paper_1502_00355_b200.distributed, with the
oracle restatement as the per-partition pass (a TEST-ONLY stand-in for tsg_pass), must
reproduce the single-process reference result bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleEngine:
    """Per-partition pass with the oracle port on the local mesh (test stand-in for tsg_pass)."""

    def __init__(self, port, part):
        self.port, self.part = port, part
        self.xy = part.xy.copy()

    def run_pass(self, cfg):
        r = self.port.smooth_prepared(self.part.topo, self.part.tri, self.xy, form="a", chunks=1, max_iters=1,
                                      move_tol=0.0)
        self.xy = r.xy
        return int(r.accepted[0]), float(r.max_disp[0])

    def pack(self, buf):
        buf.numpy()[:] = self.xy[self.part.send_ids].ravel()

    def unpack(self, buf):
        self.xy[self.part.recv_ids] = buf.numpy().reshape(-1, 2)

    def owned_coords(self):
        return self.xy[self.part.owned]


def _worker(rank, world, port_num, kind, args, max_iters, move_tol, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import paper_1502_00355_b200 as ts
    from oracle import Port
    from paper_1502_00355_b200 import capi, distributed as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_num}", rank=rank, world_size=world)
    xy, tri = ts.grid_arrays(*args) if kind == "grid" else ts.delaunay_arrays(*args)
    topo = ts.topology(len(xy), tri)
    owner = D.owners_by_order(capi.hilbert_order(xy), world)
    part = D.build_partition(rank, world, owner, xy, tri, topo)
    eng = OracleEngine(Port(), part)
    ex = D.Exchanger(part, device=False)
    it, stop, acc, md = D.smooth_partitioned(eng, ex, None, max_iters, move_tol, ts.bbox_diagonal(xy))
    full = D.gather_coords(part, eng.owned_coords(), len(xy))
    if rank == 0:
        np.savez(out_path, xy=full, acc=np.array(acc), md=np.array(md), it=it, stop=stop)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,args,tol", [
    (2, "delaunay", (3000, 5), 0.0),
    (3, "grid", (37, 41, 0.3, 2), 1e-6),
    (2, "delaunay", (800, 9), 1e-4),
])
def test_partitioned_equals_single_process(tmp_path, port, world, kind, args, tol):
    import paper_1502_00355_b200 as ts

    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), kind, args, 40, tol, out), nprocs=world, join=True)
    r = np.load(out)
    xy, tri = ts.grid_arrays(*args) if kind == "grid" else ts.delaunay_arrays(*args)
    want = port.smooth(xy, tri, form="a", chunks=1, max_iters=40, move_tol=tol)
    assert int(r["it"]) == want.iterations and str(r["stop"]) == want.stop
    assert np.array_equal(r["acc"], want.accepted)
    assert np.array_equal(r["md"].view(np.uint64), want.max_disp.view(np.uint64))
    assert np.array_equal(r["xy"].view(np.uint64), want.xy.view(np.uint64))


def test_partition_invariants():
    import paper_1502_00355_b200 as ts
    from paper_1502_00355_b200 import capi, distributed as D

    xy, tri = ts.delaunay_arrays(5000, 3)
    topo = ts.topology(len(xy), tri)
    world = 4
    owner = D.owners_by_order(capi.hilbert_order(xy), world)
    parts = [D.build_partition(r, world, owner, xy, tri, topo) for r in range(world)]
    assert sum(p.n_owned for p in parts) == len(xy)
    for p in parts:
        # every movable owned vertex has its full one-ring locally
        movable = (p.topo["boundary"] == 0)
        assert np.array_equal(np.diff(p.topo["nbr_off"])[movable],
                              np.diff(np.asarray(topo["nbr_off"]))[p.gids[movable]])
        # halo is pinned
        assert (p.topo["boundary"][~p.owned] == 1).all()
        # my recv counts from q == q's send counts to me, same vertices (by global id)
        for q in parts:
            if q.rank == p.rank:
                continue
            a = p.gids[p.recv_ids[sum(p.recv_counts[:q.rank]):sum(p.recv_counts[:q.rank + 1])]]
            b = q.gids[q.send_ids[sum(q.send_counts[:p.rank]):sum(q.send_counts[:p.rank + 1])]]
            assert np.array_equal(a, b)


def _worker_files(rank, world, port_num, part_dir, max_iters, move_tol, out_path):
    """Per-rank prep: rank 0 prepared the partition files; this rank loads only its own."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    from oracle import Port
    from paper_1502_00355_b200 import distributed as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_num}", rank=rank, world_size=world)
    part, meta = D.load_partition(part_dir, rank)
    eng = OracleEngine(Port(), part)
    ex = D.Exchanger(part, device=False)
    it, stop, acc, md = D.smooth_partitioned(eng, ex, None, max_iters, move_tol, meta["bbox_diag"])
    full = D.gather_coords(part, eng.owned_coords(), meta["nv"])
    if rank == 0:
        np.savez(out_path, xy=full, acc=np.array(acc), md=np.array(md), it=it, stop=stop)
    dist.destroy_process_group()


@pytest.mark.parametrize("weighted", [False, True])
def test_eight_ranks_from_partition_files(tmp_path, port, weighted):
    """8 ranks, each loading only its partition file (distributed.write_partitions /
    load_partition), Hilbert ranges by vertex count or by row work (1 + valence, the graded
    mesh's hubs): bit-identical to the single-process reference result."""
    import paper_1502_00355_b200 as ts
    from paper_1502_00355_b200 import capi, distributed as D

    world = 8
    xy, tri = ts.graded_arrays(6000, 5, 4e-3, 256)
    topo = ts.topology(len(xy), tri)
    order = capi.hilbert_order(xy)
    if weighted:
        owner = D.owners_by_weight(order, 1 + np.diff(topo["nbr_off"]), world)
    else:
        owner = D.owners_by_order(order, world)
    assert set(np.unique(owner)) == set(range(world))
    part_dir = str(tmp_path / "parts")
    D.write_partitions(part_dir, world, owner, xy, tri, topo, ts.bbox_diagonal(xy))
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker_files, args=(world, _free_port(), part_dir, 25, 1e-6, out), nprocs=world, join=True)
    r = np.load(out)
    want = port.smooth(xy, tri, form="a", chunks=1, max_iters=25, move_tol=1e-6)
    assert int(r["it"]) == want.iterations and str(r["stop"]) == want.stop
    assert np.array_equal(r["acc"], want.accepted)
    assert np.array_equal(r["xy"].view(np.uint64), want.xy.view(np.uint64))


def test_owners_by_weight_balances_work():
    from paper_1502_00355_b200 import distributed as D

    rng = np.random.default_rng(3)
    w = rng.integers(1, 6, size=10000).astype(np.float64)
    w[rng.integers(0, 10000, size=20)] = 1000.0  # hubs
    order = rng.permutation(10000)
    owner = D.owners_by_weight(order, w, 4)
    loads = np.bincount(owner, weights=w, minlength=4)
    assert loads.max() - loads.min() <= 2 * w.max()
    # contiguous in the order
    assert np.all(np.diff(owner[order]) >= 0)
