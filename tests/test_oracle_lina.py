"""Pins of the LinA oracle (oracle/lina.py; ADER-DG-SEM acoustics on cuboids)
against closed forms and independent constructions: Gauss-Lobatto quadrature exactness,
exact differentiation of polynomials, the weak-form stiffness by an independent Gauss rule
and numpy Lagrange fits, the upwind split of the homogeneous Riemann problem, interface
continuity of the Godunov state, the steady constant state (divergence theorem), linearity
and plane-wave convergence at order N+1 (as P:1269-1272 validates SeisSol)."""
import numpy as np
import pytest
from scipy.special import roots_legendre

from oracle import lina


@pytest.mark.parametrize("N", [1, 2, 3, 5, 7])
def test_gll_rule(N):
    x, w, *_ = lina.matrices(N)
    assert x[0] == 0.0 and x[-1] == 1.0 and np.all(np.diff(x) > 0)
    assert np.allclose(x + x[::-1], 1.0, atol=1e-15)  # symmetric
    for k in range(2 * N):  # exact to degree 2N-1
        assert abs((w * x ** k).sum() - 1.0 / (k + 1)) < 1e-14
    assert abs((w * x ** (2 * N)).sum() - 1.0 / (2 * N + 1)) > 1e-12  # Lobatto, not Gauss


@pytest.mark.parametrize("N", [1, 3, 7])
def test_derivative_matrix_is_exact_on_polynomials(N):
    x, w, Kt, Kh, Fh = lina.matrices(N)
    for k in range(N + 1):
        want = -k * x ** (k - 1) if k else np.zeros_like(x)
        assert np.abs(Kt @ x ** k - want).max() < 1e-12 * max(1, k * N * N)


def _lagrange_coeffs(x):
    """Monomial coefficients of the Lagrange polynomials on x (numpy fits, independent)."""
    n = len(x)
    return [np.polynomial.polynomial.polyfit(x, np.eye(n)[i], n - 1) for i in range(n)]


@pytest.mark.parametrize("N", [2, 4, 7])
def test_weak_stiffness_by_independent_quadrature(N):
    """Kh_kl = (1/w_k) int_0^1 psi'_k psi_l (reading L5), by a 2N-point Gauss-Legendre rule."""
    x, w, Kt, Kh, Fh = lina.matrices(N)
    g, gw = roots_legendre(2 * N)
    g, gw = (g + 1) / 2, gw / 2
    P = np.polynomial.polynomial
    c = _lagrange_coeffs(x)
    psi = np.array([P.polyval(g, ci) for ci in c])
    dpsi = np.array([P.polyval(g, P.polyder(ci)) for ci in c])
    want = (dpsi * gw) @ psi.T / w[:, None]
    assert np.abs(Kh - want).max() < 1e-10 * np.abs(want).max()
    assert Fh[0, 0] == -1 / w[0] and Fh[1, N] == -1 / w[N] and np.count_nonzero(Fh) == 2


@pytest.mark.parametrize("axis,sign", [(0, 1.0), (1, -1.0), (2, 1.0)])
def test_flux_homogeneous_upwind_and_interface_conditions(axis, sign):
    rho, K = 1800.0, 4.5e9
    Ap, Am = lina.flux_solvers(axis, sign, (rho, K), (rho, K))
    An = sign * lina.jacobians(rho, K)[axis]
    lam, X = np.linalg.eig(An)
    absA = (X @ np.diag(np.abs(lam)) @ np.linalg.inv(X)).real
    scale = np.abs(An).max()
    assert np.abs(Ap - 0.5 * (An + absA)).max() < 1e-9 * scale
    assert np.abs(Am - 0.5 * (An - absA)).max() < 1e-9 * scale
    # heterogeneous: consistency and continuity of (p*, u_n*) seen from both sides
    m1, m2 = (1500.0, 2.2e9), (2600.0, 9.0e9)
    Ap, Am = lina.flux_solvers(axis, sign, m1, m2)
    An1 = sign * lina.jacobians(*m1)[axis]
    assert np.abs(Ap + Am - An1).max() < 1e-12 * np.abs(An1).max()
    rng = np.random.default_rng(axis)
    q1, q2 = rng.standard_normal(4) * [1e6, 1, 1, 1], rng.standard_normal(4) * [1e6, 1, 1, 1]
    F12 = Ap @ q1 + Am @ q2                                   # side 1, normal n
    Bp, Bm = lina.flux_solvers(axis, -sign, m2, m1)
    F21 = Bp @ q2 + Bm @ q1                                   # side 2, normal -n
    # F = (K u_n*, p* n / rho): recover p* and u_n* on both sides
    n = np.zeros(3)
    n[axis] = sign
    p1, u1 = F12[1:] @ n * m1[0], F12[0] / m1[1]
    p2, u2 = -(F21[1:] @ n) * m2[0], F21[0] / m2[1]
    assert abs(p1 - p2) < 1e-9 * abs(p1) and abs(u1 + u2) < 1e-9 * max(1.0, abs(u1))


def _grid(N, n, hetero=True, seed=0):
    rng = np.random.default_rng(seed)
    E = n ** 3
    if hetero:
        mat = np.stack([rng.uniform(1000, 3000, E), rng.uniform(1e9, 1e10, E)], 1)
    else:
        mat = np.tile([2000.0, 8e9], (E, 1))
    return lina.setup(N, n, n, n, (1.0 / n,) * 3, mat), mat


def test_constant_state_is_steady():
    g, _ = _grid(3, 3, hetero=False)
    n = g.N + 1
    Q = np.zeros((g.E, n, n, n, 4))
    Q[...] = [3.0e5, 0.7, -1.1, 0.4]
    c = np.sqrt(8e9 / 2000.0)
    dt = 0.1 / 3 / c
    I, Ds = lina.time_integral(g, Q, dt)
    # D^1 of a constant vanishes (rows of Kt sum to zero up to rounding)
    assert np.abs(Ds[1]).max() < 1e-14 * np.abs(g.Kt).max() * np.abs(g.Astar).max() * 3e5
    vol = lina._apply3(g.Kh, I, g.Astar)
    out = lina.update(g, Q, I)
    assert np.abs(vol).max() > 1e3  # the volume terms that the fluxes cancel are large
    assert np.abs(out - Q).max() < 1e-12 * np.abs(vol).max()


def test_linearity():
    g, _ = _grid(2, 3)
    rng = np.random.default_rng(1)
    shp = (g.E, 3, 3, 3, 4)
    Q1, Q2 = rng.uniform(-1, 1, shp), rng.uniform(-1, 1, shp)
    dt = 1e-5
    lhs = lina.step(g, 0.3 * Q1 - 2.0 * Q2, dt)
    rhs = 0.3 * lina.step(g, Q1, dt) - 2.0 * lina.step(g, Q2, dt)
    assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(lhs).max()


def _plane_wave_error(N, n):
    rho, K = 2000.0, 8e9
    c, Z = np.sqrt(K / rho), np.sqrt(K * rho)
    g, _ = _grid(N, n, hetero=False)
    k = 2 * np.pi * np.array([1.0, 1.0, 0.0])
    khat = k / np.linalg.norm(k)
    om = c * np.linalg.norm(k)
    x = g.nodes
    e = np.arange(g.E)
    i, j, l = e % n, (e // n) % n, e // (n * n)
    X = (i[:, None, None, None] + x[None, :, None, None]) / n
    Y = (j[:, None, None, None] + x[None, None, :, None]) / n
    Zc = (l[:, None, None, None] + x[None, None, None, :]) / n
    X, Y, Zc = np.broadcast_arrays(X, Y, Zc)

    def exact(t):
        ph = np.sin(k[0] * X + k[1] * Y + k[2] * Zc - om * t)
        return np.stack([Z * ph, khat[0] * ph, khat[1] * ph, khat[2] * ph], -1)

    T = 0.25 * 2 * np.pi / om
    steps = 4 * n
    Q = lina.step(g, exact(0.0), T / steps, steps)
    w3 = g.w[:, None, None] * g.w[None, :, None] * g.w[None, None, :]
    scale = np.array([Z, 1, 1, 1])
    err = np.sqrt((w3[None, ..., None] * ((Q - exact(T)) / scale) ** 2).sum())
    ref = np.sqrt((w3[None, ..., None] * (exact(T) / scale) ** 2).sum())
    return err / ref


@pytest.mark.parametrize("N", [2, 3])
def test_plane_wave_convergence_order(N):
    """4^3 -> 8^3 elements: rates 2.79 (N = 2) and 3.90 (N = 3); N = 1 is pre-asymptotic at
    these sizes (1.58) and is not asserted."""
    e1, e2 = _plane_wave_error(N, 4), _plane_wave_error(N, 8)
    rate = np.log2(e1 / e2)
    assert rate > N + 1 - 0.35, (e1, e2, rate)
