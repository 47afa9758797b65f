"""Multi-rank host logic of the z-slab decomposition, world size 2 (and 3) over gloo on CPU.

Each rank builds its halo plan with the library's host-only ``ydg_halo_plan`` (the same
code ``ydg_set_comm`` + ``ydg_upload_mesh`` run), fills the send buffer with per-element
"traces" (a function of the global element id), exchanges them with gloo send/recv exactly
as the NCCL group in ``Halo::exchange`` does (one message per peer), and checks that every
ghost slot received the right element's data and that every off-rank neighbour of an owned
element is a ghost.  No GPU kernels are involved (those ranks cannot be emulated on one GPU).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

VALS = 5  # values per element "trace" in this test


def _fake_trace(gids):
    g = np.asarray(gids, dtype=np.float64)[:, None]
    return g * 10.0 + np.arange(VALS)[None, :]


def _worker(rank, world, port, nx, nz, out):
    import torch
    import paper_1903_11521_b200 as ydg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        xyz, vid = synth.kuhn_mesh(nx, nx, nz)
        ne = vid.shape[0]
        plan = ydg.ydg_halo_plan(vid, rank, world)
        first, last = ne * rank // world, ne * (rank + 1) // world
        assert (plan["send_elem"] >= first).all() and (plan["send_elem"] < last).all()
        send = torch.from_numpy(_fake_trace(plan["send_elem"]))
        recv = torch.zeros((len(plan["ghost_of"]), VALS), dtype=torch.float64)
        reqs = []
        so = ro = 0
        for k, peer in enumerate(plan["peers"]):
            sc, rc = int(plan["send_cnt"][k]), int(plan["recv_cnt"][k])
            reqs.append(dist.isend(send[so:so + sc].contiguous(), int(peer)))
            buf = torch.zeros((rc, VALS), dtype=torch.float64)
            reqs.append((dist.irecv(buf, int(peer)), buf, ro))
            so += sc
            ro += rc
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                recv[r[2]:r[2] + r[1].shape[0]] = r[1]
            else:
                r.wait()
        ok_data = bool(np.array_equal(recv.numpy(), _fake_trace(plan["ghost_of"])))
        # completeness: every off-rank neighbour of an owned element is a ghost
        from oracle import mesh as omesh
        nb = omesh.match_faces(vid)
        off = {int(n) for e in range(first, last) for n in nb[e] if not (first <= n < last)}
        ok_cover = off == set(int(g) for g in plan["ghost_of"])
        out[rank] = (ok_data, ok_cover, len(plan["ghost_of"]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,nx,nz", [(2, 3, 4), (3, 3, 6), (2, 4, 2)])
def test_halo_plan_exchange_gloo(world, nx, nz):
    import paper_1903_11521_b200 as ydg
    if not os.path.exists(ydg.LIB_PATH):
        pytest.skip("libydg.so not built")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), nx, nz, out), nprocs=world, start_method="spawn")
    for r in range(world):
        ok_data, ok_cover, ng = out[r]
        assert ok_data and ok_cover and ng > 0, (r, out[r])


def test_single_rank_plan_is_empty():
    import paper_1903_11521_b200 as ydg
    if not os.path.exists(ydg.LIB_PATH):
        pytest.skip("libydg.so not built")
    xyz, vid = synth.kuhn_mesh(3, 3, 3)
    plan = ydg.ydg_halo_plan(vid, 0, 1)
    assert len(plan["peers"]) == 0 and len(plan["ghost_of"]) == 0
