"""Pins of the oracle's ADER-DG step (oracle/step.py) against what the paper and the
mathematics fix: steady constant states (divergence theorem), polynomial termination of
the CK recursion, linearity, the paper's literal factored
Einstein sums, plane-wave convergence at order N+1 and the
viscoelastic closed forms of reading R14."""
from math import comb, factorial

import numpy as np
import pytest

import synth
from oracle import matrices, mesh, step
from tests import quadrature as qd


def _problem(cfg, P=9, Yzero=False, homogeneous=False):
    xyz, vid = synth.kuhn_mesh(cfg.nx, cfg.ny, cfg.nz, seed=cfg.seed)
    mat = synth.material(cfg)
    if homogeneous:
        mat = np.tile(mat[0], (mat.shape[0], 1))
    omega = Y = None
    if P == 27:
        omega, Y = synth.anelastic(cfg, mat)
        if Yzero:
            Y = np.zeros_like(Y)
    return step.setup(cfg.N, xyz, vid, mat, P=P, omega=omega, Y=Y), xyz, vid, mat


C0 = synth.CONFIGS["c0"]
SMALL = C0.replica(3, name="c0-r3")


def test_constant_state_is_steady():
    prob, *_ = _problem(C0)
    rng = np.random.default_rng(0)
    Q = np.zeros((C0.n_elements, comb(C0.N + 3, 3), 9))
    Q[:, 0, :] = rng.uniform(-1, 1, 9)
    I, Ds = step.time_integral(prob, Q, C0.dt)
    assert np.abs(Ds[1]).max() == 0.0  # D^1 = 0 for a constant
    vol = sum(np.einsum("kl,elq->ekq", prob.Kh[c], I) @ np.transpose(prob.Astar[:, c], (0, 2, 1)) for c in range(3))
    Q1 = step.update(prob, Q, I)
    assert np.abs(vol).max() > 1e3  # the terms that must cancel are large
    assert np.abs(Q1 - Q).max() < 1e-13 * np.abs(vol).max()


@pytest.mark.parametrize("N", [2, 5])
def test_derivative_recursion_terminates_on_data(N):
    cfg = SMALL.__class__(**{**SMALL.__dict__, "N": N})
    prob, *_ = _problem(cfg)
    Q = step.to_internal(synth.dofs(cfg))
    I, Ds = step.time_integral(prob, Q, cfg.dt)
    for d, D in enumerate(Ds):
        rows = comb(N - d + 3, 3)
        assert not D[:, rows:, :].any()  # staircase
    # one more derivative is exactly zero
    Dn = sum(np.einsum("kl,elq->ekq", prob.Kt[c], Ds[-1]) @ np.transpose(prob.Astar[:, c], (0, 2, 1)) for c in range(3))
    assert np.abs(Dn).max() == 0.0


def test_linearity():
    prob, *_ = _problem(SMALL)
    rng = np.random.default_rng(1)
    Q1 = step.to_internal(synth.dofs(SMALL))
    Q2 = rng.uniform(-1, 1, Q1.shape)
    a, b = 0.7, -1.9
    lhs = step.step(prob, a * Q1 + b * Q2, SMALL.dt)
    rhs = a * step.step(prob, Q1, SMALL.dt) + b * step.step(prob, Q2, SMALL.dt)
    assert np.abs(lhs - rhs).max() < 1e-13 * np.abs(lhs).max()


@pytest.mark.parametrize("N", [1, 2])
def test_literal_einsum_matches(N):
    cfg = SMALL.__class__(**{**SMALL.__dict__, "N": N})
    prob, xyz, vid, mat = _problem(cfg)
    Q = step.to_internal(synth.dofs(cfg))
    dense = step.step(prob, Q, cfg.dt)
    lit = step.literal_update(prob, Q, cfg.dt, mesh.neighbour_table(vid))
    assert np.abs(dense - lit).max() < 1e-14 * np.abs(dense).max()


def _project(N, xyz, func):
    """L2 projection of func(x) (npts,3)->(npts,9) on every element: Q (E, B, 9)."""
    pts, w = qd.tet_rule(N + 3)
    phi = matrices.basis_eval(N, pts)
    x = xyz[:, 0, None, :] + np.einsum("rc,ecd->erd", pts, np.stack([xyz[:, 1] - xyz[:, 0], xyz[:, 2] - xyz[:, 0], xyz[:, 3] - xyz[:, 0]], 1))
    vals = func(x.reshape(-1, 3)).reshape(x.shape[0], len(w), 9)
    return np.einsum("rk,r,erp->ekp", phi, w, vals), (pts, w, phi, x)


def _plane_wave_error(N, n, nsteps_per_n=4):
    rho, vp = 2500.0, 5000.0
    vs = vp / np.sqrt(3.0)
    from oracle import physics
    lam, mu = physics.lame(rho, vp, vs)
    A = physics.jacobians(rho, lam, mu)
    k = 2 * np.pi / n * np.array([1.0, 1.0, 0.0])
    Ak = np.einsum("d,dpq->pq", k, A)
    w, X = np.linalg.eig(Ak)
    idx = np.argmax(w.real)
    omega, r = w[idx].real, X[:, idx].real
    r = r / np.abs(r).max()

    def exact(x, t):
        return np.sin(x @ k - omega * t)[:, None] * r[None, :]

    xyz, vid = synth.kuhn_mesh(n, n, n, seed=3)
    E = xyz.shape[0]
    mat = np.tile([rho, vp, vs], (E, 1))
    prob = step.setup(N, xyz, vid, mat)
    Q, (pts, wq, phi, x) = _project(N, xyz, lambda y: exact(y, 0.0))
    period = 2 * np.pi / omega
    T = 0.2 * period
    nsteps = nsteps_per_n * n
    Q = step.step(prob, Q, T / nsteps, nsteps)
    qh = np.einsum("rk,ekp->erp", phi, Q)
    qe = exact(x.reshape(-1, 3), T).reshape(qh.shape)
    detJ = mesh.geometry(xyz)[2]
    # stresses (~Z v) and velocities differ by ~1e7: weigh each group by its amplitude
    scale = np.r_[np.full(6, np.abs(r[:6]).max()), np.full(3, np.abs(r[6:]).max())][None, None, :]
    err = np.sqrt((detJ[:, None, None] * wq[None, :, None] * ((qh - qe) / scale) ** 2).sum())
    ref = np.sqrt((detJ[:, None, None] * wq[None, :, None] * (qe / scale) ** 2).sum())
    return err / ref


@pytest.mark.parametrize("N", [1, 2])
def test_plane_wave_convergence_order(N):
    """the observed convergence order matches the theoretical order N+1."""
    e4 = _plane_wave_error(N, 4)
    e8 = _plane_wave_error(N, 8)
    rate = np.log2(e4 / e8)
    assert rate > N + 1 - 0.3, (e4, e8, rate)


def test_visco_Y_zero_reduces_to_elastic():
    cfg = SMALL.__class__(**{**SMALL.__dict__, "N": 2, "P": 27})
    prob27, *_ = _problem(cfg, P=27, Yzero=True)
    prob9, *_ = _problem(cfg, P=9)
    Q27 = step.to_internal(synth.dofs(cfg))
    out27 = step.step(prob27, Q27, cfg.dt)
    out9 = step.step(prob9, np.ascontiguousarray(Q27[:, :, :9]), cfg.dt)
    assert np.abs(out27[:, :, :9] - out9).max() < 1e-13 * np.abs(out9).max()


def test_visco_constant_state_is_truncated_exponential():
    # homogeneous material: every element relaxes with the same E, so the state stays constant
    cfg = SMALL.__class__(**{**SMALL.__dict__, "N": 3, "P": 27})
    prob, *_ = _problem(cfg, P=27, homogeneous=True)
    rng = np.random.default_rng(2)
    q0 = rng.uniform(-1, 1, 27)
    Q = np.zeros((cfg.n_elements, comb(cfg.N + 3, 3), 27))
    Q[:, 0, :] = q0
    out = step.step(prob, Q, cfg.dt)
    for e in [0, 7, 100]:
        Et = prob.E_src[e].T * cfg.dt
        S = np.zeros((27, 27))
        term = np.eye(27)
        for kk in range(cfg.N + 2):
            S += term / factorial(kk)
            term = term @ Et
        want = q0 @ S
        assert np.abs(out[e, 0] - want).max() < 1e-12 * np.abs(want).max() + 1e-9
        assert np.abs(out[e, 1:]).max() < 1e-9 * np.abs(want).max()


def test_fused_simulations_equal_independent_runs():
    """S fused simulations (extra index s on Q, D, I; all matrices shared) are S
    independent runs of the single-simulation scheme."""
    prob, *_ = _problem(SMALL)
    rng = np.random.default_rng(5)
    S = 3
    Qs = rng.uniform(-1, 1, (S, SMALL.n_elements, comb(SMALL.N + 3, 3), 9))
    fused = step.step_fused(prob, Qs, SMALL.dt, 2)
    for s in range(S):
        single = step.step(prob, Qs[s], SMALL.dt, 2)
        assert np.abs(fused[s] - single).max() <= 1e-13 * np.abs(single).max()
    # the simulations do not mix: a zero simulation stays zero
    Qs[1] = 0.0
    assert not step.step_fused(prob, Qs, SMALL.dt, 1)[1].any()
