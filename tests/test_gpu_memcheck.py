"""Out-of-bounds and race checks of the CUDA path (compute-sanitizer substitutes).

compute-sanitizer is not allowed on this GPU pool, so the kernels are checked
with the library's own instruments:

* guard zones (``YDG_GUARD=1``): every device buffer of the mesh and the DOFs gets 64 KiB of
  a fill pattern on both sides; after the steps ``ydg_query(YDG_Q_GUARD_VIOLATIONS)`` must
  report no overwritten guard byte (an out-of-bounds global store of any kernel family
  lands in a guard zone of its buffer or its neighbour's);
* race check: the persistent kernels assign tiles to work groups by the grid size, and the
  work groups of one CTA share shared memory, fragment buffers and named barriers, so the
  results of the same input under other grid sizes (``YDG_GRID_LOCAL`` / ``YDG_GRID_NEIGH``,
  one virtual CTA up to several per SM) and on a repeated run must be bitwise identical --
  a missing barrier or a shared-memory race shows up as a difference.
"""
import numpy as np
import pytest

import synth
from tests.helpers import make_inputs

pytestmark = pytest.mark.gpu


def _run(cfg, nsteps, env, monkeypatch, sims=1, lts=False):
    import paper_1903_11521_b200 as ydg
    for k in ("YDG_GUARD", "YDG_GRID_LOCAL", "YDG_GRID_NEIGH"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    xyz, vid, mat, Q, an = make_inputs(cfg)
    h = ydg.ydg_create(cfg.N, cfg.P, cfg.precision)
    try:
        if sims > 1:
            ydg.ydg_set_simulations(h, sims)
        if lts:
            # two clusters: the coarse cluster is the first half of the elements, rounded
            # to whole tiles (ydg_set_clusters' contract)
            tw = int(ydg.ydg_query(h, ydg.YDG_Q_TILE_ELEMENTS))
            cl = np.zeros(len(vid), np.int8)
            cl[: (len(vid) // 2) // tw * tw] = 1
            ydg.ydg_set_clusters(h, cl)
        ydg.ydg_upload_mesh(h, xyz, vid, mat, an)
        n = int(ydg.ydg_query(h, ydg.YDG_Q_N_ELEMENTS))
        rng = np.random.default_rng(7)
        Qs = np.concatenate([Q] * sims) if sims > 1 else Q
        Qs = (Qs * (1.0 + 0.1 * rng.standard_normal(Qs.shape))).astype(h.dtype)
        ydg.ydg_upload_dofs(h, 0, Qs[:n])
        guard0 = ydg.ydg_query(h, ydg.YDG_Q_GUARD_VIOLATIONS)
        if lts:
            ydg.ydg_step_lts(h, cfg.dt, nsteps)
        else:
            ydg.ydg_step(h, cfg.dt, nsteps)
        out = ydg.ydg_download_dofs(h, 0, n)
        guard1 = ydg.ydg_query(h, ydg.YDG_Q_GUARD_VIOLATIONS)
    finally:
        ydg.ydg_destroy(h)
    return out, guard0, guard1


CASES = {
    "fp64-N5-vperm": (synth.CONFIGS["c1"].replica(4).with_(vperm=True, name="c1-vperm"), 2, {}),
    "fp64-N2-ragged": (synth.CONFIGS["c0"].with_(N=2, nx=3, ny=3, nz=3, vperm=True, name="r"), 2, {}),
    "fp32-N6": (synth.CONFIGS["c2"].replica(3, steps=2).with_(vperm=True, name="c2-vperm"), 2, {}),
    "visco-N4": (synth.CONFIGS["c3"].replica(3).with_(vperm=True, name="c3-vperm"), 2, {}),
    "generic-fp64-N6": (synth.CONFIGS["c0"].with_(N=6, nx=3, ny=3, nz=3, vperm=True, name="g6"), 1, {}),
    "fused-sims-4": (synth.CONFIGS["c0"].with_(N=3, vperm=True, name="s4"), 2, {"sims": 4}),
    "lts-N3": (synth.CONFIGS["c0"].with_(N=3, nx=4, ny=4, nz=4, vperm=True, name="lts"), 2, {"lts": True}),
}


@pytest.mark.parametrize("name", list(CASES))
def test_guard_zones_intact(name, monkeypatch):
    """No kernel of the case writes outside its buffers (guard zones intact)."""
    cfg, nsteps, kw = CASES[name]
    out, g0, g1 = _run(cfg, nsteps, {"YDG_GUARD": "1"}, monkeypatch, **kw)
    print(f"{name}: guard violations before {g0:.0f}, after {g1:.0f}; max|Q| {np.abs(out).max():.3e}")
    assert g0 == 0 and g1 == 0
    assert np.isfinite(out).all()


def test_guard_query_without_guards(monkeypatch):
    cfg = synth.CONFIGS["c0"].with_(N=1, name="c0-n1")
    _, g0, g1 = _run(cfg, 1, {}, monkeypatch)
    assert g0 == -1 and g1 == -1


GRIDS = [{}, {}, {"YDG_GRID_LOCAL": "1", "YDG_GRID_NEIGH": "1"},
         {"YDG_GRID_LOCAL": "7", "YDG_GRID_NEIGH": "5"}, {"YDG_GRID_LOCAL": "37", "YDG_GRID_NEIGH": "301"}]


@pytest.mark.parametrize("name", ["fp64-N5-vperm", "fp32-N6", "visco-N4", "fused-sims-4", "lts-N3"])
def test_bitwise_under_grid_sizes(name, monkeypatch):
    """Repeated runs and other persistent grid sizes give bitwise identical results."""
    cfg, nsteps, kw = CASES[name]
    outs = [_run(cfg, nsteps, env, monkeypatch, **kw)[0] for env in GRIDS]
    for env, o in zip(GRIDS[1:], outs[1:]):
        same = np.array_equal(o.view(np.uint8), outs[0].view(np.uint8))
        assert same, (name, env, np.abs(o - outs[0]).max())


@pytest.mark.parametrize("name", ["fp64-N2-ragged", "fp32-N6", "visco-N4", "generic-fp64-N6", "fused-sims-4"])
def test_max_abs_q_diagnostic(name, monkeypatch):
    """ydg_query(YDG_Q_MAX_ABS_Q) (the per-step max|Q| diagnostic of SURVEY §5) equals the
    maximum of the downloaded DOFs exactly, and turns NaN when one DOF is not finite."""
    import paper_1903_11521_b200 as ydg
    cfg, nsteps, kw = CASES[name]
    sims = kw.get("sims", 1)
    for k in ("YDG_GUARD", "YDG_GRID_LOCAL", "YDG_GRID_NEIGH"):
        monkeypatch.delenv(k, raising=False)
    xyz, vid, mat, Q, an = make_inputs(cfg)
    h = ydg.ydg_create(cfg.N, cfg.P, cfg.precision)
    try:
        if sims > 1:
            ydg.ydg_set_simulations(h, sims)
        ydg.ydg_upload_mesh(h, xyz, vid, mat, an)
        n = int(ydg.ydg_query(h, ydg.YDG_Q_N_ELEMENTS))
        Qs = (np.concatenate([Q] * sims) if sims > 1 else Q).astype(h.dtype)[:n]
        ydg.ydg_upload_dofs(h, 0, Qs)
        assert ydg.ydg_query(h, ydg.YDG_Q_MAX_ABS_Q) == float(np.abs(Qs).max())
        ydg.ydg_step(h, cfg.dt, nsteps)
        out = ydg.ydg_download_dofs(h, 0, n)
        assert ydg.ydg_query(h, ydg.YDG_Q_MAX_ABS_Q) == float(np.abs(out).max())
        bad = out[n // 2: n // 2 + 1].copy()
        bad[0, 1, 2] = np.nan
        ydg.ydg_upload_dofs(h, n // 2, bad)
        assert np.isnan(ydg.ydg_query(h, ydg.YDG_Q_MAX_ABS_Q))
    finally:
        ydg.ydg_destroy(h)
