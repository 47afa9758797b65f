"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerances (BASELINE.json north_star): max|dQ| / max|Q| <= 1e-12 in fp64, <= 2e-5 in fp32;
neighbour / face / orientation tables bit-exact.
"""
import numpy as np
import pytest

import synth
from oracle import mesh as omesh
from tests.helpers import LAST_PATH, TOL, check_parity, face_cases, make_inputs, rel_err, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def _cfg(name, **kw):
    base = synth.CONFIGS[name]
    return base.__class__(**{**base.__dict__, **kw})


def _parity(cfg, nsteps=None, dt=None, check=True):
    xyz, vid, mat, Q, an = make_inputs(cfg)
    got, nbt = run_gpu(cfg, xyz, vid, mat, Q, an, nsteps=nsteps, dt=dt)
    ref = run_oracle(cfg, xyz, vid, mat, Q, an, nsteps=nsteps, dt=dt)
    err = rel_err(got, ref)
    if check:
        check_parity(err, cfg.precision, cfg.name)
    return err, nbt, vid


def test_c0_parity_and_tables():
    """BASELINE configs[0]: full mesh, 1 step, fp64."""
    cfg = synth.CONFIGS["c0"]
    err, (nb, j, h), vid = _parity(cfg)
    onb, oj, oh = omesh.neighbour_table(vid)
    assert np.array_equal(nb, onb) and np.array_equal(j, oj) and np.array_equal(h, oh)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_orders_fp64_ragged(N):
    """3x3x3 cubes = 162 elements: 20 full 8-element tiles (fp64) and a ragged tail of 2."""
    cfg = _cfg("c0", N=N, nx=3, ny=3, nz=3)
    err, *_ = _parity(cfg, nsteps=2)


def test_c1_replica_fp64():
    """configs[1] at 8x8x8 cubes (3072 elements), N=5, fp64, its 10 steps (SURVEY §8(c)
    parity protocol 2)."""
    cfg = synth.CONFIGS["c1"].replica(8)
    err, *_ = _parity(cfg)


def test_c2_replica_fp32():
    """configs[2] at 8x8x8 cubes, N=6, fp32, two-layer material, 6 of its 10 steps: the
    config's dt (0.2 h / vp_max, reading R13) is 2-6x the ADER-DG CFL bound, so max|Q| grows
    ~700x per step (oracle: 3.9e9 after 1 step, 2.7e23 after 6, 8.8e34 after 10) and the
    fp32 intermediates of steps 9-10 reach FLT_MAX; 6 steps is the longest run whose fp32
    values are all far from overflow."""
    cfg = synth.CONFIGS["c2"].replica(8, steps=6)
    err, *_ = _parity(cfg)


# ---- unstructured neighbour relations: every (face i, neighbour face j, orientation h)
# case of Neigh/Face/Rot.  The Kuhn order alone yields 6 of the 48 cases; a
# per-element random even vertex permutation (synth vperm) yields all of them, as the
# paper's reproducer's random neighbour relations do.

def _perm_parity(cfg, nsteps=None, dt=None):
    err, (nb, j, h), vid = _parity(cfg, nsteps=nsteps, dt=dt)
    assert len(face_cases(vid)) == 48
    onb, oj, oh = omesh.neighbour_table(vid)
    assert np.array_equal(nb, onb) and np.array_equal(j, oj) and np.array_equal(h, oh)
    return err


def test_vperm_c0_fp64():
    _perm_parity(synth.CONFIGS["c0"].with_(vperm=True, name="c0-vperm"))


@pytest.mark.parametrize("N", [1, 3, 4])
def test_vperm_orders_fp64(N):
    _perm_parity(synth.CONFIGS["c0"].with_(N=N, nx=3, ny=3, nz=3, vperm=True, name=f"N{N}-vperm"), nsteps=2)


def test_vperm_c1_replica_fp64():
    _perm_parity(synth.CONFIGS["c1"].replica(6, steps=3).with_(vperm=True, name="c1-vperm"))


def test_vperm_c2_replica_fp32():
    _perm_parity(synth.CONFIGS["c2"].replica(6, 6, 4, steps=2).with_(vperm=True, name="c2-vperm"))


def test_vperm_c3_viscoelastic():
    _perm_parity(synth.CONFIGS["c3"].replica(4, 4, 3, steps=2).with_(vperm=True, name="c3-vperm"))
    assert LAST_PATH["path"] == 2


def test_vperm_generic(monkeypatch):
    monkeypatch.setenv("YDG_GENERIC", "1")
    _perm_parity(synth.CONFIGS["c0"].with_(vperm=True, name="generic-vperm"), nsteps=2)


def test_vperm_order6_fp64_generic():
    _perm_parity(synth.CONFIGS["c1"].with_(N=6, nx=3, ny=3, nz=3, steps=1, vperm=True, name="N6-vperm"))


def test_vperm_visco_generic(monkeypatch):
    monkeypatch.setenv("YDG_VISCO_GENERIC", "1")
    _perm_parity(synth.CONFIGS["c3"].replica(3, steps=1).with_(vperm=True, name="c3csr-vperm"))
    assert LAST_PATH["path"] == 3


def test_fp32_at_stable_dt():
    """fp32 at a stable time step (reading R13) so growth cannot hide precision loss."""
    cfg = _cfg("c0", precision=4, N=4, nx=3, ny=3, nz=3)
    err, *_ = _parity(cfg, nsteps=5, dt=0.02 / 6000.0)


def test_constant_state_is_steady_on_gpu():
    import paper_1903_11521_b200 as ydg
    cfg = synth.CONFIGS["c0"]
    xyz, vid, mat, Q, _ = make_inputs(cfg)
    Qc = np.zeros_like(Q)
    Qc[:, :, 0] = np.linspace(-1, 1, 9)[None, :]
    h = ydg.ydg_create(cfg.N, 9, 8)
    ydg.ydg_upload_mesh(h, xyz, vid, mat)
    ydg.ydg_upload_dofs(h, 0, Qc)
    ydg.ydg_step(h, cfg.dt, 1)
    out = ydg.ydg_download_dofs(h, 0, len(Q))
    # the volume and face terms that cancel are ~1e6 here (lambda dt |Q| / h): 1e-8 absolute
    # is ~1e-14 relative; several steps at the (unstable, reading R13) config dt amplify
    # the rounding noise, so one step is checked
    assert np.abs(out - Qc).max() < 1e-7  # the oracle gives 1.02e-8 on the same input


def test_errors_and_state():
    import paper_1903_11521_b200 as ydg
    with pytest.raises(ydg.YdgError):
        ydg.ydg_create(0, 9, 8)
    with pytest.raises(ydg.YdgError):
        ydg.ydg_create(3, 10, 8)
    h = ydg.ydg_create(2, 9, 8)
    with pytest.raises(ydg.YdgError) as ei:
        ydg.ydg_step(h, 1e-4, 1)
    assert ei.value.code == ydg.YDG_ERR_STATE
    xyz, vid = synth.kuhn_mesh(3, 3, 3)
    mat = synth.material(synth.CONFIGS["c0"].replica(3))
    with pytest.raises(ydg.YdgError) as ei:
        ydg.ydg_upload_mesh(h, xyz[:-1], vid[:-1], mat[:-1])  # open mesh
    assert ei.value.code == ydg.YDG_ERR_MESH
    bad = xyz.copy()
    bad[0, [1, 2]] = bad[0, [2, 1]]  # det J < 0
    with pytest.raises(ydg.YdgError) as ei:
        ydg.ydg_upload_mesh(h, bad, vid, mat)
    assert ei.value.code == ydg.YDG_ERR_MESH
    ydg.ydg_upload_mesh(h, xyz, vid, mat)
    with pytest.raises(ydg.YdgError) as ei:
        ydg.ydg_download_dofs(h, 100, 1000)
    assert ei.value.code == ydg.YDG_ERR_ARG
    # zero steps is a no-op; empty transfers are allowed
    ydg.ydg_step(h, 1e-4, 0)
    ydg.ydg_download_dofs(h, 0, 0)
    ydg.ydg_destroy(h)


def test_c3_viscoelastic_replica():
    """configs[3] (viscoelastic, 3 mechanisms, P = 27, N = 4, fp64) at 3x3x3 cubes, 2 steps:
    generic CUDA path vs the oracle of reading R14."""
    cfg = synth.CONFIGS["c3"].replica(3, steps=2)
    err, *_ = _parity(cfg)
    assert LAST_PATH["path"] == 2  # the viscoelastic tensor-core kernels ran


@pytest.mark.parametrize("N", [1, 2, 3])
def test_viscoelastic_orders(N):
    """The viscoelastic tensor-core local kernel at the other orders it is generated for
    (3x3x2 cubes: 108 elements = 13 full 8-element tiles + a ragged tile of 4)."""
    cfg = _cfg("c3", N=N, nx=3, ny=3, nz=2, steps=2)
    err, *_ = _parity(cfg)
    assert LAST_PATH["path"] == 2


def test_viscoelastic_csr_kernel(monkeypatch):
    """YDG_VISCO_GENERIC=1 selects the CSR local kernel (the comparison path); it agrees too."""
    monkeypatch.setenv("YDG_VISCO_GENERIC", "1")
    cfg = synth.CONFIGS["c3"].replica(3, steps=1)
    err, *_ = _parity(cfg)
    assert LAST_PATH["path"] == 3


def test_generic_path_elastic(monkeypatch):
    """The generic (CSR) kernels on the elastic c0 problem agree with the oracle too."""
    monkeypatch.setenv("YDG_GENERIC", "1")
    err, *_ = _parity(synth.CONFIGS["c0"], nsteps=2)


def test_order6_fp64_generic():
    cfg = _cfg("c1", N=6, nx=3, ny=3, nz=3, steps=1)
    err, *_ = _parity(cfg)


def test_viscoelastic_order5_generic():
    """P = 27 at N = 5 runs the CSR kernels with 2-element CTAs (4 do not fit in 227 KB)."""
    cfg = synth.CONFIGS["c3"].with_(N=5, nx=3, ny=3, nz=2, steps=1, vperm=True, name="c3-N5")
    _parity(cfg)
    assert LAST_PATH["path"] == 3


def test_generic_handles_of_both_quantity_counts_coexist(monkeypatch):
    """A P = 9 and a P = 27 generic handle alive in one process, steps interleaved: each keeps
    its own star / source column patterns."""
    import paper_1903_11521_b200 as ydg
    monkeypatch.setenv("YDG_GENERIC", "1")
    monkeypatch.setenv("YDG_VISCO_GENERIC", "1")
    c9 = synth.CONFIGS["c0"].with_(nx=3, ny=3, nz=3, name="coexist-9")
    c27 = synth.CONFIGS["c3"].with_(N=2, nx=3, ny=3, nz=3, steps=1, name="coexist-27")
    ins = {c.name: make_inputs(c) for c in (c9, c27)}
    hs = {}
    for c in (c9, c27):  # P = 9 first: the later P = 27 configuration must not clobber it
        xyz, vid, mat, Q, an = ins[c.name]
        h = ydg.ydg_create(c.N, c.P, c.precision)
        ydg.ydg_upload_mesh(h, xyz, vid, mat, an)
        ydg.ydg_upload_dofs(h, 0, Q)
        hs[c.name] = h
    for c in (c9, c27, c9):
        ydg.ydg_step(hs[c.name], c.dt, 1)
    for c, n in ((c9, 2), (c27, 1)):
        got = ydg.ydg_download_dofs(hs[c.name], 0, c.n_elements)
        ref = run_oracle(c, *ins[c.name], nsteps=n)
        check_parity(rel_err(got, ref), 8, c.name)
        ydg.ydg_destroy(hs[c.name])


def test_step_graph_matches_step():
    """ydg_step_graph (the nsteps launch sequence as one CUDA graph) is bitwise ydg_step, and
    is re-captured when dt changes."""
    import paper_1903_11521_b200 as ydg
    cfg = synth.CONFIGS["c0"]
    xyz, vid, mat, Q, _ = make_inputs(cfg)
    outs = []
    for graph in (False, True):
        h = ydg.ydg_create(cfg.N, 9, 8)
        ydg.ydg_upload_mesh(h, xyz, vid, mat)
        ydg.ydg_upload_dofs(h, 0, Q)
        f = ydg.ydg_step_graph if graph else ydg.ydg_step
        f(h, cfg.dt, 3)
        f(h, cfg.dt, 3)
        f(h, 0.5 * cfg.dt, 3)
        outs.append(ydg.ydg_download_dofs(h, 0, cfg.n_elements))
        ydg.ydg_destroy(h)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("S,prec", [(4, 8), (16, 8), (8, 4)])
def test_fused_simulations(S, prec):
    """NEXT-1: S fused simulations (element-simulations v = e*S + s, adjacent
    lanes of a tile) against the oracle's scheme with the index s; neighbours Neigh(e,i)*S+s."""
    import paper_1903_11521_b200 as ydg
    from oracle import step as ostep
    cfg = synth.CONFIGS["c0"].with_(vperm=True, precision=prec, name=f"fused-S{S}")
    xyz, vid, mat, _, _ = make_inputs(cfg)
    E = cfg.n_elements
    Qs = synth.uniform(cfg.seed + 1, synth.STREAM_DOFS, np.arange(S * E * 9 * cfg.B, dtype=np.uint64), -1, 1)
    Qs = Qs.reshape(S, E, 9, cfg.B)  # [s][e][p][k]
    h = ydg.ydg_create(cfg.N, 9, prec)
    ydg.ydg_set_simulations(h, S)
    ydg.ydg_upload_mesh(h, xyz, vid, mat)
    assert ydg.ydg_query(h, ydg.YDG_Q_N_ELEMENTS) == S * E
    assert ydg.ydg_query(h, ydg.YDG_Q_SIMULATIONS) == S
    dt_np = np.float64 if prec == 8 else np.float32
    ydg.ydg_upload_dofs(h, 0, np.ascontiguousarray(Qs.transpose(1, 0, 2, 3)).reshape(E * S, 9, cfg.B).astype(dt_np))
    ydg.ydg_step(h, cfg.dt, 2)
    got = ydg.ydg_download_dofs(h, 0, E * S).reshape(E, S, 9, cfg.B).transpose(1, 0, 2, 3).astype(np.float64)
    nb, j, hr = ydg.ydg_get_neighbours(h, 0, E * S)
    ydg.ydg_destroy(h)
    onb, oj, oh = omesh.neighbour_table(vid)
    v = np.arange(E * S)
    assert np.array_equal(nb, onb[v // S] * S + (v % S)[:, None])
    assert np.array_equal(j, oj[v // S]) and np.array_equal(hr, oh[v // S])
    prob = ostep.setup(cfg.N, xyz, vid, mat)
    ref = ostep.step_fused(prob, np.ascontiguousarray(Qs.transpose(0, 1, 3, 2)), cfg.dt, 2).transpose(0, 1, 3, 2)
    for s in range(S):
        check_parity(rel_err(got[s], ref[s]), prec, f"fused S={S} s={s}")


def _lts_clusters(cfg, xyz):
    """Elements of the upper half (centroid z >= nz/2) coarse: whole z-layers of cubes, so
    the coarse count is a multiple of the tile width."""
    return (xyz[:, :, 2].mean(1) >= cfg.nz / 2).astype(np.int8)


@pytest.mark.parametrize("N,vperm", [(2, False), (5, True), (3, True)])
def test_local_time_stepping(N, vperm):
    """NEXT-2 (reading R26): two-cluster LTS cycles on the GPU (ydg_step_lts) against the
    oracle's LTS (oracle/lts.py), including the cluster interface in both directions."""
    import paper_1903_11521_b200 as ydg
    from oracle import lts as olts
    from oracle import step as ostep
    cfg = synth.CONFIGS["c0"].with_(N=N, nx=4, ny=4, nz=4, vperm=vperm, name=f"lts-N{N}")
    xyz, vid, mat, Q, _ = make_inputs(cfg)
    cl = _lts_clusters(cfg, xyz)
    assert cl.sum() % 16 == 0 and 0 < cl.sum() < len(cl)
    dt = cfg.dt / 4
    h = ydg.ydg_create(cfg.N, 9, 8)
    ydg.ydg_set_clusters(h, cl)
    ydg.ydg_upload_mesh(h, xyz, vid, mat)
    ydg.ydg_upload_dofs(h, 0, Q)
    ydg.ydg_step_lts(h, dt, 2)
    got = ydg.ydg_download_dofs(h, 0, cfg.n_elements)
    nb, j, hr = ydg.ydg_get_neighbours(h, 0, cfg.n_elements)
    ydg.ydg_destroy(h)
    onb, oj, oh = omesh.neighbour_table(vid)
    assert np.array_equal(nb, onb) and np.array_equal(j, oj) and np.array_equal(hr, oh)
    prob = ostep.setup(cfg.N, xyz, vid, mat)
    ref = ostep.to_canonical(olts.lts(prob, ostep.to_internal(Q), dt, cl, 2))
    check_parity(rel_err(got, ref), 8, cfg.name)


def test_lts_rejects_ragged_coarse_cluster():
    import paper_1903_11521_b200 as ydg
    cfg = synth.CONFIGS["c0"]
    xyz, vid, mat, Q, _ = make_inputs(cfg)
    cl = np.zeros(cfg.n_elements, np.int8)
    cl[:5] = 1
    h = ydg.ydg_create(cfg.N, 9, 8)
    ydg.ydg_set_clusters(h, cl)
    with pytest.raises(ydg.YdgError) as ei:
        ydg.ydg_upload_mesh(h, xyz, vid, mat)
    assert ei.value.code == ydg.YDG_ERR_ARG
    ydg.ydg_destroy(h)


@pytest.mark.parametrize("N,cubes,vperm", [(2, 3, True), (3, 3, True), (5, 4, True), (5, 6, False)])
def test_fused_step_kernel_is_bitwise_two_kernel_steps(monkeypatch, N, cubes, vperm):
    """With YDG_FUSED=1, ydg_step(nsteps >= 2) on one rank runs the fused kernel (the flux of step n-1, then the
    local part of step n, per tile; traces in two alternating buffers).  It performs the same
    operations in the same order as the two-kernel steps (YDG_FUSED=0), so the results are
    bitwise equal -- over calls of 1, 2 and 5 steps, on meshes with every (i, j, h) face case
    and a ragged last tile -- and match the oracle."""
    import paper_1903_11521_b200 as ydg
    cfg = synth.CONFIGS["c0"].with_(N=N, nx=cubes, ny=cubes, nz=cubes, vperm=vperm, name=f"fused-N{N}")
    xyz, vid, mat, Q, _ = make_inputs(cfg)
    outs = []
    for fz in ("1", "0"):
        monkeypatch.setenv("YDG_FUSED", fz)
        h = ydg.ydg_create(cfg.N, 9, 8)
        ydg.ydg_upload_mesh(h, xyz, vid, mat)
        assert ydg.ydg_query(h, ydg.YDG_Q_FUSED) == (1.0 if fz == "1" else 0.0)
        ydg.ydg_upload_dofs(h, 0, Q)
        for n in (1, 2, 5):
            ydg.ydg_step(h, cfg.dt, n)
        outs.append(ydg.ydg_download_dofs(h, 0, cfg.n_elements))
        ydg.ydg_destroy(h)
    assert np.array_equal(outs[0], outs[1])
    ref = run_oracle(cfg, xyz, vid, mat, Q, nsteps=8)
    check_parity(rel_err(outs[0], ref), 8, cfg.name)


def test_fused_kernel_grid_sizes_bitwise(monkeypatch):
    """The fused kernel's persistent grid (work groups walking tiles) does not change the
    result: 1, 7 and 592 groups, bitwise."""
    import paper_1903_11521_b200 as ydg
    cfg = synth.CONFIGS["c0"].with_(N=5, nx=4, ny=4, nz=4, vperm=True, name="fused-grid")
    xyz, vid, mat, Q, _ = make_inputs(cfg)
    outs = []
    monkeypatch.setenv("YDG_FUSED", "1")
    for g in ("1", "7", "592"):
        monkeypatch.setenv("YDG_GRID_LOCAL", g)
        h = ydg.ydg_create(cfg.N, 9, 8)
        ydg.ydg_upload_mesh(h, xyz, vid, mat)
        assert ydg.ydg_query(h, ydg.YDG_Q_FUSED) == 1.0
        ydg.ydg_upload_dofs(h, 0, Q)
        ydg.ydg_step(h, cfg.dt, 4)
        outs.append(ydg.ydg_download_dofs(h, 0, cfg.n_elements))
        ydg.ydg_destroy(h)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("N,prec", [(5, 8), (2, 8), (6, 4), (3, 4)])
def test_accounting_queries(N, prec):
    """The bench's roofline inputs: the per-kernel nonzero flops add up to the canonical count
    of the step (both flux terms with their own lifts), the executed flux count
    (one lift per face) is below it by the local lifts, and the algorithmic bytes per
    element follow the arrays each kernel touches once (written out here from the layouts)."""
    import paper_1903_11521_b200 as ydg
    cfg = synth.CONFIGS["c0"].with_(N=N, precision=prec, name=f"acct-N{N}")
    xyz, vid, mat, Q, _ = make_inputs(cfg)
    h = ydg.ydg_create(N, 9, prec)
    ydg.ydg_upload_mesh(h, xyz, vid, mat)
    q = lambda k: ydg.ydg_query(h, k)
    B, Bt, P = (N + 1) * (N + 2) * (N + 3) // 6, (N + 1) * (N + 2) // 2, 9
    assert q(ydg.YDG_Q_B) == B and q(ydg.YDG_Q_BTILDE) == Bt
    nz, loc, nb, nbx = (q(ydg.YDG_Q_NZ_FLOPS), q(ydg.YDG_Q_LOCAL_FLOPS), q(ydg.YDG_Q_NEIGH_FLOPS),
                        q(ydg.YDG_Q_NEIGH_FLOPS_EXEC))
    assert loc + nb == nz
    # one lift per face instead of two: the executed flux count drops by 4 * 9 * nnz(R) FMAs
    # of the local lifts (2 flops each) -- the same R^i appear in both lifts
    assert 0 < nbx < nb
    by_l, by_n = q(ydg.YDG_Q_LOCAL_BYTES), q(ydg.YDG_Q_NEIGH_BYTES)
    assert q(ydg.YDG_Q_ALG_BYTES) == by_l + by_n
    # star matrices as stored: 3 directions x 9 rows x 3 columns per element
    if prec == 4:  # fp32 tiled kernels: traces [m][q] per face, 9x9 A+ and A- per face
        assert by_l == (2 * B * P + 81 + 4 * Bt * P) * 4
        assert by_n == (2 * B * P + 8 * P * P + 8 * Bt * P) * 4 + 20
    else:  # fp64: element-face trace blocks of TS = even(9 Bt) doubles, 12 flux coefficients
        TS = (9 * Bt + 1) // 2 * 2
        assert by_l == (2 * B * P + 81 + 4 * TS) * 8
        assert by_n == (2 * B * P + 48 + 8 * TS) * 8 + 20
        assert q(ydg.YDG_Q_FUSED_BYTES) == (2 * B * P + 81 + 48 + 12 * TS) * 8 + 20
    ydg.ydg_destroy(h)
