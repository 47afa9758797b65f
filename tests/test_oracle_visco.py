"""Independent pins of the oracle's viscoelastic parts (reading R14 / SURVEY §8(c) C14).

The paper only cites viscoelasticity; the equations are reading R14:
    d_t sigma - C_u : eps(v) = - sum_l Y_l : theta^l,   (Y:th)_ij = Ylam tr(th) d_ij + 2 Ymu th_ij
    rho d_t v - div sigma = 0
    d_t theta^l - omega_l eps(v) = - omega_l theta^l,    eps = sym grad v
None of the pins below reuses the oracle's E or Jacobians to build its expected value:
* the source matrix against the (Y:theta) table written out for unit tensors;
* D^1 of a linear velocity field (sigma = theta = 0) against the continuum right-hand side
  omega_l sym(G), lam tr(G) I + mu (G + G^T), 0 -- this fixes the 1/2 of the tensor strain
  rate, the sign and the omega_l of the memory-variable Jacobian rows;
* a theta-only constant state against the scalar closed form of the truncated Taylor
  series of d_t theta = -omega theta, d_t sigma = -Y:theta (no matrix exponential);
* the plane-wave dispersion relation rho s^2 + k^2 M(s) = 0 with the relaxation moduli
  M(s) = M_u - sum_l Y^M_l omega_l / (s + omega_l), derived from the equations above by a
  Laplace transform, against the eigenvalues of E - i k A_x;
* rotational invariance A_n = T A_x T^-1 and T T^-1 = I for P = 27 (memory tensors rotate
  like stresses), flux consistency A+ + A- = A_n(m-) including the memory rows.
"""
from math import comb, factorial

import numpy as np
import pytest

import synth
from oracle import matrices, mesh, physics, step
from tests import quadrature as qd

VOIGT = ((0, 0), (1, 1), (2, 2), (0, 1), (1, 2), (0, 2))


def _yl_table(Ylam, Ymu):
    """6 x 6 block: d_t sigma (rows, Voigt) from a unit memory tensor component (columns).
    Column xx: theta = e_x e_x^T -> Y:theta = Ylam I + 2 Ymu e_x e_x^T; column xy: theta_xy =
    theta_yx = 1 -> Y:theta has 2 Ymu in xy (tr = 0)."""
    a, b = Ylam + 2 * Ymu, Ylam
    return -np.array([
        [a, b, b, 0, 0, 0],
        [b, a, b, 0, 0, 0],
        [b, b, a, 0, 0, 0],
        [0, 0, 0, 2 * Ymu, 0, 0],
        [0, 0, 0, 0, 2 * Ymu, 0],
        [0, 0, 0, 0, 0, 2 * Ymu],
    ])


def test_source_matrix_against_unit_tensor_table():
    omega = np.array([0.3, 2.0, 17.0])
    Ylam = np.array([1.5e8, 2.5e8, 3.5e8])
    Ymu = np.array([0.7e8, 1.1e8, 1.3e8])
    E = physics.source_matrix(omega, Ylam, Ymu)
    want = np.zeros((27, 27))
    for l in range(3):
        c = slice(9 + 6 * l, 15 + 6 * l)
        want[0:6, c] = _yl_table(Ylam[l], Ymu[l])
        want[c, c] = -omega[l] * np.eye(6)
    assert np.array_equal(E, want)
    # velocity rows and every elastic column are source-free
    assert not E[6:9].any() and not E[:, 0:9].any()


def _project(N, xyz, func, P):
    pts, w = qd.tet_rule(N + 3)
    phi = matrices.basis_eval(N, pts)
    Jc = np.stack([xyz[:, 1] - xyz[:, 0], xyz[:, 2] - xyz[:, 0], xyz[:, 3] - xyz[:, 0]], 1)
    x = xyz[:, 0, None, :] + np.einsum("rc,ecd->erd", pts, Jc)
    vals = func(x.reshape(-1, 3)).reshape(x.shape[0], len(w), P)
    return np.einsum("rk,r,erp->ekp", phi, w, vals), phi


@pytest.mark.parametrize("N", [1, 3])
def test_linear_velocity_field_drives_memory_variables(N):
    """v(x) = G x, sigma = theta = 0: D^1 (= d_t q) is the constant continuum right-hand side."""
    cfg = synth.CONFIGS["c3"].replica(3, name="c3-r3").with_(N=N)
    xyz, vid = synth.kuhn_mesh(3, 3, 3, seed=5)
    mat = synth.material(cfg)
    omega, Y = synth.anelastic(cfg, mat)
    prob = step.setup(N, xyz, vid, mat, P=27, omega=omega, Y=Y)
    G = np.random.default_rng(11).uniform(-1, 1, (3, 3))

    def field(x):
        q = np.zeros((x.shape[0], 27))
        q[:, 6:9] = x @ G.T
        return q

    Q, phi = _project(N, xyz, field, 27)
    _, Ds = step.time_integral(prob, Q, cfg.dt)
    rate = np.einsum("rk,ekp->erp", phi, Ds[1])  # d_t q at the quadrature points
    lam, mu = physics.lame(mat[:, 0], mat[:, 1], mat[:, 2])
    eps = 0.5 * (G + G.T)
    for e in (0, 17, 100):
        want = np.zeros(27)
        S = lam[e] * np.trace(G) * np.eye(3) + 2 * mu[e] * eps
        for v, (i, j) in enumerate(VOIGT):
            want[v] = S[i, j]
            for l in range(3):
                want[9 + 6 * l + v] = omega[l] * eps[i, j]
        err = np.abs(rate[e] - want[None, :]).max(axis=0)
        assert err[:6].max() <= 1e-12 * np.abs(want[:6]).max(), (e, err[:6])
        assert err[6:9].max() <= 1e-12 * np.abs(want[:6]).max() / mat[e, 0], (e, err[6:9])
        assert err[9:].max() <= 1e-12 * np.abs(want[9:]).max(), (e, err[9:])


@pytest.mark.parametrize("N", [2, 4])
def test_memory_only_constant_state_decays_by_truncated_exponential(N):
    """sigma = v = 0, theta^l = c_l constant, homogeneous material.  Then I (and the update)
    follow from scalars: theta^l(dt) = c_l sum_{k<=N+1} (-omega_l dt)^k / k!,
    sigma(dt) = sum_l Y_l : c_l / omega_l * sum_{1<=k<=N+1} (-omega_l dt)^k / k!."""
    cfg = synth.CONFIGS["c3"].replica(3, name="c3-r3").with_(N=N)
    xyz, vid = synth.kuhn_mesh(3, 3, 3, seed=cfg.seed)
    mat = np.tile(synth.material(cfg)[0], (cfg.n_elements, 1))
    omega, Y = synth.anelastic(cfg, mat)
    omega = np.array([30.0, 700.0, 9000.0])  # large enough that dt omega matters
    prob = step.setup(N, xyz, vid, mat, P=27, omega=omega, Y=Y)
    rng = np.random.default_rng(3)
    c = rng.uniform(-1, 1, (3, 6))
    Q = np.zeros((cfg.n_elements, comb(N + 3, 3), 27))
    for l in range(3):
        Q[:, 0, 9 + 6 * l:15 + 6 * l] = c[l]
    dt = 1e-4
    out = step.step(prob, Q, dt)
    want = np.zeros(27)
    for l in range(3):
        x = -omega[l] * dt
        want[9 + 6 * l:15 + 6 * l] = c[l] * sum(x ** k / factorial(k) for k in range(N + 2))
        g = sum(x ** k / factorial(k) for k in range(1, N + 2)) / omega[l]
        th = np.zeros((3, 3))
        for v, (i, j) in enumerate(VOIGT):
            th[i, j] = th[j, i] = c[l, v]
        S = Y[0, l, 0] * np.trace(th) * np.eye(3) + 2 * Y[0, l, 1] * th
        for v, (i, j) in enumerate(VOIGT):
            want[v] += S[i, j] * g
    got = out[:, 0, :] * 1.0
    assert np.abs(got[:, 6:9]).max() < 1e-12  # no velocity is generated
    for e in (0, 50, 161):
        assert np.abs(got[e, :6] - want[:6]).max() <= 1e-12 * np.abs(want[:6]).max()
        assert np.abs(got[e, 9:] - want[9:]).max() <= 1e-13
    assert np.abs(out[:, 1:, :]).max() <= 1e-9 * np.abs(want[:6]).max()  # stays constant


def _dispersion_roots(rho, M, YM, omega, k):
    """Roots s of rho s^2 prod(s + w_l) + k^2 (M prod(s + w_l) - sum_l YM_l w_l prod_{m!=l}(s + w_m))."""
    prod = np.poly1d([1.0])
    for w in omega:
        prod = prod * np.poly1d([1.0, w])
    poly = np.poly1d([rho, 0.0, 0.0]) * prod + k * k * M * prod
    for l, w in enumerate(omega):
        others = np.poly1d([1.0])
        for m, w2 in enumerate(omega):
            if m != l:
                others = others * np.poly1d([1.0, w2])
        poly = poly - k * k * YM[l] * w * others
    return poly.roots


def test_plane_wave_dispersion_relation():
    rho, lam, mu = 1.3, 2.1, 0.9
    omega = np.array([0.5, 1.7, 4.0])
    Ylam, Ymu = np.array([0.11, 0.07, 0.05]), np.array([0.06, 0.04, 0.09])
    k = 1.3
    A = physics.jacobians(rho, lam, mu, 27, omega)
    E = physics.source_matrix(omega, Ylam, Ymu)
    # q = qh exp(i k x + s t):  s qh = (E - i k A_x) qh
    ev = np.linalg.eigvals(E - 1j * k * A[0])
    p_roots = _dispersion_roots(rho, lam + 2 * mu, Ylam + 2 * Ymu, omega, k)
    s_roots = _dispersion_roots(rho, mu, Ymu, omega, k)  # sigma_xy = 2 mu eps_xy, eps_xy = i k v_y / 2
    for r in p_roots:
        assert np.abs(ev - r).min() < 1e-8 * max(1.0, abs(r)), ("P", r)
    for r in s_roots:  # two shear polarisations
        d = np.sort(np.abs(ev - r))
        assert d[1] < 1e-6 * max(1.0, abs(r)), ("S", r, d[:3])
    # the remaining 12 eigenvalues are the uncoupled relaxations -omega_l and zeros
    rest = list(ev)
    for r in list(p_roots) + list(s_roots) + list(s_roots):
        rest.pop(int(np.argmin(np.abs(np.array(rest) - r))))
    allowed = np.r_[0.0, -omega]
    assert all(np.abs(allowed - r).min() < 1e-6 for r in rest)


def test_rotation_of_memory_tensors():
    rng = np.random.default_rng(8)
    n = rng.standard_normal(3)
    n /= np.linalg.norm(n)
    R = physics.face_frame(n)
    T, Ti = physics.rotation(R, 27), physics.rotation(R.T, 27)
    assert np.abs(T @ Ti - np.eye(27)).max() < 1e-14
    # a memory tensor rotates like the stress: S_g = R S_f R^T, for every mechanism slot
    q = rng.standard_normal(27)
    g = T @ q
    for base in (0, 9, 15, 21):
        S = np.zeros((3, 3))
        for v, (i, j) in enumerate(VOIGT):
            S[i, j] = S[j, i] = q[base + v]
        Sg = R @ S @ R.T
        assert np.allclose([Sg[i, j] for (i, j) in VOIGT], g[base:base + 6], atol=1e-14)
    # rotational invariance of the viscoelastic system: A_n = T A_x T^-1
    omega = np.array([0.6, 6.0, 60.0])
    A = physics.jacobians(2500.0, 3e10, 2e10, 27, omega)
    An = np.einsum("d,dpq->pq", n, A)
    assert np.abs(T @ A[0] @ Ti - An).max() < 1e-9 * np.abs(An).max()


def test_viscoelastic_flux_consistency():
    rng = np.random.default_rng(9)
    n = rng.standard_normal(3)
    n /= np.linalg.norm(n)
    omega = np.array([0.6, 6.0, 60.0])
    m1 = (2100.0,) + physics.lame(2100.0, 3300.0, 3300.0 / np.sqrt(3))
    m2 = (2900.0,) + physics.lame(2900.0, 5800.0, 5800.0 / np.sqrt(3))
    Ap, Am = physics.flux_solvers(n, m1, m2, 27, omega)
    An = np.einsum("d,dpq->pq", n, physics.jacobians(*m1, 27, omega))
    assert np.abs(Ap + Am - An).max() < 1e-12 * np.abs(An).max()
    # memory-variable columns never enter the Riemann problem
    assert not Ap[:, 9:].any() and not Am[:, 9:].any()
    # memory rows = -omega_l x the velocity part of eps(v*): ratio of mechanisms is omega
    assert np.allclose(Ap[15:21] * omega[0], Ap[9:15] * omega[1], atol=1e-12 * np.abs(Ap[9:15]).max())


def test_match_faces_subset_agrees_with_full_matching():
    xyz, vid = synth.kuhn_mesh(4, 3, 3, vperm=True)
    full = mesh.match_faces(vid)
    sel = np.array([0, 5, 77, 100, len(vid) - 1])
    assert np.array_equal(step._match_faces_subset(vid, sel), full[sel])
    assert np.array_equal(step._match_faces_subset(vid, np.arange(len(vid))), full)
