"""Partition invariance of the z-slab decomposition: P ranks (loopback halo
transport: handles of one process, one host thread each, on one GPU; same halo plan, pack,
ghost slots and unpack as the NCCL path) produce Q bitwise identical to one rank."""
import os
import threading

import numpy as np
import pytest

import synth
from tests.helpers import make_inputs

pytestmark = pytest.mark.gpu


def _run(cfg, nranks, nsteps):
    import paper_1903_11521_b200 as ydg
    xyz, vid, mat, Q, an = make_inputs(cfg)
    Q = Q.astype(np.float64 if cfg.precision == 8 else np.float32)
    uid = b"YDGLOOP" + os.urandom(16) + bytes(128 - 23)
    parts, errors = [None] * nranks, []

    def work(r):
        try:
            h = ydg.ydg_create(cfg.N, cfg.P, cfg.precision, device=0)
            if nranks > 1:
                ydg.ydg_set_comm(h, r, nranks, uid)
            ydg.ydg_upload_mesh(h, xyz, vid, mat, an)
            first = int(ydg.ydg_query(h, ydg.YDG_Q_FIRST_LOCAL))
            n = int(ydg.ydg_query(h, ydg.YDG_Q_N_LOCAL))
            ydg.ydg_upload_dofs(h, first, Q[first:first + n])
            ydg.ydg_step(h, cfg.dt, nsteps)
            parts[r] = (first, ydg.ydg_download_dofs(h, first, n))
            ydg.ydg_destroy(h)
        except Exception as ex:  # noqa: BLE001 -- reported below
            errors.append(ex)

    threads = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=240)
    assert not errors, errors
    out = np.empty_like(Q)
    for first, q in parts:
        out[first:first + len(q)] = q
    return out


@pytest.mark.parametrize("nranks", [2, 4])
def test_zslab_partition_is_bitwise_invariant(nranks):
    """c1 replica (N = 5, fp64) on 8x8x8 cubes, 3 steps: P-rank result == 1-rank result."""
    cfg = synth.CONFIGS["c1"].replica(8, steps=3)
    ref = _run(cfg, 1, cfg.steps)
    got = _run(cfg, nranks, cfg.steps)
    assert np.array_equal(got, ref), np.abs(got - ref).max()


def test_zslab_partition_fp32():
    cfg = synth.CONFIGS["c2"].replica(6, 6, 4, steps=2)
    ref = _run(cfg, 1, cfg.steps)
    got = _run(cfg, 2, cfg.steps)
    assert np.array_equal(got, ref), np.abs(got - ref).max()


def test_c4_replica_eight_ranks():
    """BASELINE configs[4] shape (N = 5 fp64, strong scaling over z-slabs) on an 8x8x16-cube
    replica split into 8 slabs of 2 cube layers (every element touches a slab boundary side),
    random neighbour relations (vperm): bitwise the 1-rank result."""
    cfg = synth.CONFIGS["c4"].replica(8, 8, 16, steps=2).with_(vperm=True)
    ref = _run(cfg, 1, cfg.steps)
    got = _run(cfg, 8, cfg.steps)
    assert np.array_equal(got, ref), np.abs(got - ref).max()


def test_reordered_elements_are_bitwise_invariant(monkeypatch):
    """YDG_REORDER=1 (Morton / boundary-first internal order) changes no result bit, on one
    rank and on 3 ranks."""
    cfg = synth.CONFIGS["c1"].replica(6, steps=2).with_(vperm=True)
    ref = _run(cfg, 1, cfg.steps)
    monkeypatch.setenv("YDG_REORDER", "1")
    assert np.array_equal(_run(cfg, 1, cfg.steps), ref)
    assert np.array_equal(_run(cfg, 3, cfg.steps), ref)
