"""Multi-rank host logic of the z-slab decomposition, world size 2 (and 3) over gloo on CPU.

Each rank builds its halo plan with the library's host-only ``ydg_halo_plan`` (the same
code ``ydg_set_comm`` + ``ydg_upload_mesh`` run), fills the send buffer with per-face-block
"traces" (a function of the sending element's global id and local face), exchanges them
with gloo send/recv exactly as the NCCL group in ``Halo::exchange`` does (one message per
peer), and checks that every received block is the one the plan says (element, face), that
these are exactly the shared faces every owned element's neighbour flux reads (nb, j of
P:1342 from the oracle's brute-force table) and that every off-rank neighbour is a ghost.
No GPU kernels are involved (those ranks cannot be emulated on one GPU).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

VALS = 5  # values per element "trace" in this test


def _fake_trace(gids, faces):
    g = np.asarray(gids, dtype=np.float64)[:, None] * 4 + np.asarray(faces, dtype=np.float64)[:, None]
    return g * 10.0 + np.arange(VALS)[None, :]


def _worker(rank, world, port, nx, nz, out):
    import torch
    import paper_1903_11521_b200 as ydg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        xyz, vid = synth.kuhn_mesh(nx, nx, nz, vperm=True)
        ne = vid.shape[0]
        plan = ydg.ydg_halo_plan(vid, rank, world)
        first, last = ne * rank // world, ne * (rank + 1) // world
        assert (plan["send_elem"] >= first).all() and (plan["send_elem"] < last).all()
        send = torch.from_numpy(_fake_trace(plan["send_elem"], plan["send_face"]))
        recv = torch.zeros((len(plan["recv_elem"]), VALS), dtype=torch.float64)
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
        ok_data = bool(np.array_equal(recv.numpy(), _fake_trace(plan["recv_elem"], plan["recv_face"])))
        # completeness: the received blocks are exactly the (Neigh, Face) pairs of the owned
        # elements' off-rank faces, each once; every off-rank neighbour is a ghost
        from oracle import mesh as omesh
        nb, j, _ = omesh.neighbour_table(vid)
        need = sorted((int(nb[e, i]), int(j[e, i])) for e in range(first, last) for i in range(4)
                      if not (first <= nb[e, i] < last))
        got = sorted(zip(plan["recv_elem"].tolist(), plan["recv_face"].tolist()))
        off = {n for n, _ in need}
        ok_cover = need == got and off == set(int(g) for g in plan["ghost_of"])
        # blocks sent: our side of every off-rank face, once
        mine = sorted((e, i) for e in range(first, last) for i in range(4) if not (first <= nb[e, i] < last))
        ok_send = mine == sorted(zip(plan["send_elem"].tolist(), plan["send_face"].tolist()))
        out[rank] = (ok_data, ok_cover and ok_send, len(plan["ghost_of"]))
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
