"""GPU parity of the LinA workload (NEXT-3: ADER-DG-SEM acoustics on cuboids):
the CUDA kernels (lina_local / lina_flux through include/ydg_lina.h) against oracle/lina.py
on the same seeded inputs, per quantity (pressure and velocities separately)."""
import numpy as np
import pytest

import synth
from oracle import lina as olina

pytestmark = pytest.mark.gpu


def _run(cfg, nsteps):
    import paper_1903_11521_b200 as ydg
    mat = synth.lina_material(cfg)
    Q = synth.lina_dofs(cfg)
    h = ydg.lina_create(cfg.N)
    ydg.lina_upload_grid(h, cfg.nx, cfg.ny, cfg.nz, np.array(cfg.h), mat)
    ydg.lina_upload_dofs(h, 0, Q)
    ydg.lina_step(h, cfg.dt, nsteps)
    got = ydg.lina_download_dofs(h, 0, cfg.n_elements)
    ydg.lina_destroy(h)
    g = olina.setup(cfg.N, cfg.nx, cfg.ny, cfg.nz, cfg.h, mat)
    ref = olina.step(g, np.ascontiguousarray(Q.transpose(0, 2, 3, 4, 1)), cfg.dt, nsteps).transpose(0, 4, 1, 2, 3)
    return got, ref


def _check(got, ref, label):
    errs = {}
    for q, name in enumerate(("p", "u", "v", "w")):
        errs[name] = np.abs(got[:, q] - ref[:, q]).max() / np.abs(ref[:, q]).max()
    print(f"lina parity {label}: " + " ".join(f"{k}={v:.2e}" for k, v in errs.items()))
    assert max(errs.values()) <= 1e-12, errs


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7])
def test_lina_orders(N):
    cfg = synth.LINA_CONFIGS["lina-small"].with_(N=N, h=(1.0, 0.7, 1.3))
    got, ref = _run(cfg, 2)
    _check(got, ref, f"N={N}")


def test_lina_order8_more_elements_than_ctas():
    """N = 7 (order 8, the bench order) on 12 x 11 x 10 elements: several elements per CTA."""
    cfg = synth.LINA_CONFIGS["lina"].with_(nx=12, ny=11, nz=10, steps=3)
    got, ref = _run(cfg, 3)
    _check(got, ref, "N=7 1320 elements")


def test_lina_fullsize_sampled():
    """The bench workload itself (order 8, 64^3 cuboids, the bench's launch configuration):
    one GPU step, checked on sampled elements against the oracle on the samples and their six
    neighbours (the update of an element reads only its neighbours' side tensors)."""
    import paper_1903_11521_b200 as ydg
    cfg = synth.LINA_CONFIGS["lina"]
    mat = synth.lina_material(cfg)
    Q = synth.lina_dofs(cfg)
    h = ydg.lina_create(cfg.N)
    ydg.lina_upload_grid(h, cfg.nx, cfg.ny, cfg.nz, np.array(cfg.h), mat)
    ydg.lina_upload_dofs(h, 0, Q)
    ydg.lina_step(h, cfg.dt, 1)
    rng = np.random.default_rng(3)
    sel = np.unique(np.concatenate([rng.integers(0, cfg.n_elements, 40), [0, cfg.n_elements - 1]]))
    got = np.stack([ydg.lina_download_dofs(h, int(e), 1)[0] for e in sel])
    ydg.lina_destroy(h)
    nb = olina.neighbours(cfg.nx, cfg.ny, cfg.nz)
    union = np.unique(np.concatenate([sel, nb[sel].ravel()]))
    pos = {int(e): i for i, e in enumerate(union)}
    nodes, w, Kt, Kh, Fh = olina.matrices(cfg.N)
    U = len(union)
    Astar = np.zeros((U, 3, 4, 4))
    Ap = np.zeros((U, 6, 4, 4))
    Am = np.zeros((U, 6, 4, 4))
    nbs = np.zeros((U, 6), dtype=np.int64)
    for u, e in enumerate(union):
        J = olina.jacobians(*mat[e])
        for a in range(3):
            Astar[u, a] = J[a] / cfg.h[a]
        for s, (a, end) in enumerate(olina.SIDES):
            p, m = olina.flux_solvers(a, 1.0 if end else -1.0, mat[e], mat[nb[e, s]])
            Ap[u, s], Am[u, s] = p / cfg.h[a], m / cfg.h[a]
            nbs[u, s] = pos.get(int(nb[e, s]), u)  # only the samples' rows are used
    g = olina.Grid(cfg.N, cfg.nx, cfg.ny, cfg.nz, cfg.h, Kt, Kh, Fh, w, nodes, Astar, Ap, Am, nbs)
    Qu = np.ascontiguousarray(Q[union].transpose(0, 2, 3, 4, 1))
    I, _ = olina.time_integral(g, Qu, cfg.dt)
    ref = olina.update(g, Qu, I).transpose(0, 4, 1, 2, 3)[[pos[int(e)] for e in sel]]
    _check(got, ref, "order 8 64^3 sampled")
