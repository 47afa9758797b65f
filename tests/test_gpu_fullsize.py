"""Full-size sampled parity (BASELINE configs at their full sizes, in the launch configuration
bench.py times): the library advances the whole mesh; the oracle recomputes one step for a
sample of elements (4 contiguous blocks at seeded offsets, i.e. ragged tile positions) from
the same Q^n, using the time integrals of the samples' face neighbours.

Checked at n = 0 (Q^0 from the seeded generator) and, for c1, after `steps - 1` library steps
(Q^n of the samples and their neighbours downloaded from the device), so the last step of
the benchmarked run is covered too.
"""
import numpy as np
import pytest

import synth
from oracle import step as ostep
from tests.helpers import check_parity, rel_err

pytestmark = pytest.mark.gpu


def _samples(cfg, blocks=4, width=48, seed=7):
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, cfg.n_elements - width, size=blocks)
    return np.unique(np.concatenate([np.arange(s, s + width) for s in starts]))


def _oracle_one_step(cfg, xyz, vid, mat, an, sel, Qsel, Qnb_of):
    """One oracle step for the elements `sel` given their Q (Qsel, canonical) and a function
    returning the canonical Q of arbitrary element ids (for the neighbours)."""
    omega = Y = None
    if cfg.P == 27:
        omega, Y = an[:3], an[3:].reshape(-1, 3, 2)
    prob = ostep.setup(cfg.N, xyz, vid, mat, P=cfg.P, omega=omega, Y=Y, elements=sel)
    union = np.unique(np.concatenate([sel, prob.nb.ravel()]))
    pu = ostep.setup(cfg.N, xyz, vid, mat, P=cfg.P, omega=omega, Y=Y, elements=union)
    Iu, _ = ostep.time_integral(pu, ostep.to_internal(Qnb_of(union)), cfg.dt)
    prob.nb = np.searchsorted(union, prob.nb)
    Is, _ = ostep.time_integral(prob, ostep.to_internal(Qsel), cfg.dt)
    return ostep.to_canonical(ostep.update(prob, ostep.to_internal(Qsel), Is, Iu))


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_fullsize_sampled_one_step(name):
    import paper_1903_11521_b200 as ydg
    cfg = synth.CONFIGS[name]
    xyz, vid = synth.kuhn_mesh(cfg.nx, cfg.ny, cfg.nz, seed=cfg.seed, jitter=cfg.jitter)
    mat = synth.material(cfg)
    an = None
    if cfg.P == 27:
        omega, Y = synth.anelastic(cfg, mat)
        an = np.concatenate([omega, Y.ravel()])
    h = ydg.ydg_create(cfg.N, cfg.P, cfg.precision)
    ydg.ydg_upload_mesh(h, xyz, vid, mat, an)
    dt_np = np.float64 if cfg.precision == 8 else np.float32
    Q0 = synth.dofs(cfg).astype(dt_np)
    ydg.ydg_upload_dofs(h, 0, Q0)
    sel = _samples(cfg)

    def gpu_rows(ids):
        return np.stack([ydg.ydg_download_dofs(h, int(e), 1)[0] for e in ids]).astype(np.float64)

    # n = 0 -> 1
    ydg.ydg_step(h, cfg.dt, 1)
    got = gpu_rows(sel)
    ref = _oracle_one_step(cfg, xyz, vid, mat, an, sel, Q0[sel].astype(np.float64),
                           lambda ids: Q0[ids].astype(np.float64))
    check_parity(rel_err(got, ref), cfg.precision, f"{name} n=0")
    if name == "c1":  # last step of the benchmarked run: n = steps-1 -> steps
        ydg.ydg_step(h, cfg.dt, cfg.steps - 2)
        nb = ostep.setup(cfg.N, xyz, vid, mat, elements=sel).nb
        union = np.unique(np.concatenate([sel, nb.ravel()]))
        Qn = dict(zip(union.tolist(), gpu_rows(union)))
        ydg.ydg_step(h, cfg.dt, 1)
        got = gpu_rows(sel)
        ref = _oracle_one_step(cfg, xyz, vid, mat, an, sel, np.stack([Qn[e] for e in sel]),
                               lambda ids: np.stack([Qn[e] for e in ids]))
        check_parity(rel_err(got, ref), cfg.precision, f"{name} last step")
    ydg.ydg_destroy(h)


def test_fullsize_sampled_c4():
    """BASELINE configs[4] (12.6 M tetrahedra, N = 5, fp64) on one GPU at its full size -- the
    largest mesh the library holds (~141 GB of device memory, 64-bit tile offsets): Q^0
    uploaded in 1 M-element chunks straight from the seeded generator, one step, sampled
    one-step parity against the oracle."""
    import paper_1903_11521_b200 as ydg
    cfg = synth.CONFIGS["c4"]
    xyz, vid = synth.kuhn_mesh(cfg.nx, cfg.ny, cfg.nz, seed=cfg.seed, jitter=cfg.jitter)
    mat = synth.material(cfg)
    h = ydg.ydg_create(cfg.N, cfg.P, cfg.precision)
    ydg.ydg_upload_mesh(h, xyz, vid, mat)
    E = cfg.n_elements
    chunk = 1 << 20
    for first in range(0, E, chunk):
        ydg.ydg_upload_dofs(h, first, synth.dofs(cfg, first, min(chunk, E - first)))
    sel = _samples(cfg)
    ydg.ydg_step(h, cfg.dt, 1)
    got = np.stack([ydg.ydg_download_dofs(h, int(e), 1)[0] for e in sel])
    ydg.ydg_destroy(h)

    def q0(ids):
        return np.stack([synth.dofs(cfg, int(e), 1)[0] for e in ids])

    ref = _oracle_one_step(cfg, xyz, vid, mat, None, sel, q0(sel), q0)
    check_parity(rel_err(got, ref), cfg.precision, "c4 n=0")
