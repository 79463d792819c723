"""Partitioned multi-process smoothing through the real device path (tsg_pass / tsg_halo_pack /
tsg_halo_unpack).  The test box has one GPU, so the ranks share cuda:0 and exchange halos with
gloo over host buffers; on an 8-GPU box bench.py runs the same driver with NCCL device buffers.
Result must be bit-identical to the single-GPU / oracle run (Form A)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_num, args, layout, precision, max_iters, move_tol, out_path, driver="host"):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1502_00355_b200 as ts
    from paper_1502_00355_b200 import capi, distributed as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_num}", rank=rank, world_size=world)
    xy, tri = ts.delaunay_arrays(*args)
    topo = ts.topology(len(xy), tri)
    owner = D.owners_by_order(capi.hilbert_order(xy), world)
    part = D.build_partition(rank, world, owner, xy, tri, topo)
    ctx = capi.Context(0)
    eng = D.DeviceEngine(ctx, part, layout=layout, precision=precision)
    if driver == "host":
        ex = D.Exchanger(part, device=False)
        cfg = capi.make_cfg(form="a", strategy="fused", max_iters=max_iters)
        it, stop, acc, md = D.smooth_partitioned(eng, ex, cfg, max_iters, move_tol, ts.bbox_diagonal(xy))
    else:  # device-resident loop (tsg_dist_*), gloo through host copies
        import torch

        cfg = capi.make_cfg(form="a", strategy="fused", max_iters=max_iters, move_tol=move_tol,
                            bbox_diag=ts.bbox_diagonal(xy))
        loop = D.DeviceLoop(eng, part, device=False, torch_device=torch.device("cuda", 0), stream_ptr=ctx.stream)
        it, stop, acc, md = loop.smooth(cfg, check_every=3)
    full = D.gather_coords(part, eng.owned_coords(), len(xy))
    if rank == 0:
        np.savez(out_path, xy=full, acc=np.array(acc), md=np.array(md), it=it, stop=stop)
    eng.mesh.free()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,args,layout,tol,driver", [(2, (20000, 3), "aos", 0.0, "host"),
                                                          (3, (9000, 8), "soa", 1e-6, "host"),
                                                          (2, (20000, 3), "aos", 0.0, "device"),
                                                          (3, (9000, 8), "aos", 1e-6, "device")])
def test_partitioned_device_equals_single(tmp_path, port, world, args, layout, tol, driver):
    import paper_1502_00355_b200 as ts

    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), args, layout, "f64", 30, tol, out, driver), nprocs=world, join=True)
    r = np.load(out)
    xy, tri = ts.delaunay_arrays(*args)
    want = port.smooth(xy, tri, form="a", chunks=1, max_iters=30, move_tol=tol)
    assert int(r["it"]) == want.iterations and str(r["stop"]) == want.stop
    assert np.array_equal(r["acc"], want.accepted)
    assert np.array_equal(r["md"].view(np.uint64), want.max_disp.view(np.uint64))
    assert np.array_equal(r["xy"].view(np.uint64), want.xy.view(np.uint64))
