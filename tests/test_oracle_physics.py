"""Pins of oracle/physics.py and oracle/mesh.py against textbook facts and closed forms."""
import numpy as np
import pytest

import synth
from oracle import mesh, physics

SXX, SYY, SZZ, SXY, SYZ, SXZ, U, V, W = range(9)


def typed_jacobians(rho, lam, mu):
    """The velocity-stress Jacobians typed in entry by entry (independent of physics.py)."""
    A = np.zeros((9, 9)); B = np.zeros((9, 9)); C = np.zeros((9, 9))
    l2m = lam + 2 * mu
    A[SXX, U] = -l2m; A[SYY, U] = -lam; A[SZZ, U] = -lam; A[SXY, V] = -mu; A[SXZ, W] = -mu
    A[U, SXX] = -1 / rho; A[V, SXY] = -1 / rho; A[W, SXZ] = -1 / rho
    B[SXX, V] = -lam; B[SYY, V] = -l2m; B[SZZ, V] = -lam; B[SXY, U] = -mu; B[SYZ, W] = -mu
    B[U, SXY] = -1 / rho; B[V, SYY] = -1 / rho; B[W, SYZ] = -1 / rho
    C[SXX, W] = -lam; C[SYY, W] = -lam; C[SZZ, W] = -l2m; C[SYZ, V] = -mu; C[SXZ, U] = -mu
    C[U, SXZ] = -1 / rho; C[V, SYZ] = -1 / rho; C[W, SZZ] = -1 / rho
    return np.stack([A, B, C])


def test_jacobians_match_typed_table():
    rho, vp, vs = 2500.0, 5000.0, 5000.0 / np.sqrt(3)
    lam, mu = physics.lame(rho, vp, vs)
    assert np.array_equal(physics.jacobians(rho, lam, mu), typed_jacobians(rho, lam, mu))


def test_star_matrices_have_24_nonzeros():
    rng = np.random.default_rng(1)
    Jinv = rng.standard_normal((3, 3))
    A = physics.jacobians(2000.0, 3e10, 2e10)
    S = physics.star_matrices(Jinv, A)
    for c in range(3):
        assert (S[c] != 0).sum() == 24


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_normal_jacobian_eigenvalues(seed):
    rng = np.random.default_rng(seed)
    n = rng.standard_normal(3); n /= np.linalg.norm(n)
    rho, vp = 2300.0, 4100.0
    vs = vp / np.sqrt(3)
    lam, mu = physics.lame(rho, vp, vs)
    An = np.einsum("d,dpq->pq", n, physics.jacobians(rho, lam, mu))
    ev = np.sort(np.linalg.eigvals(An).real)
    want = np.sort([-vp, vp, -vs, -vs, vs, vs, 0, 0, 0])
    assert np.allclose(ev, want, atol=1e-6 * vp)


def test_rotation_is_consistent():
    rng = np.random.default_rng(3)
    n = rng.standard_normal(3); n /= np.linalg.norm(n)
    R = physics.face_frame(n)
    assert np.allclose(R.T @ R, np.eye(3), atol=1e-15)
    T, Ti = physics.rotation(R), physics.rotation(R.T)
    assert np.allclose(T @ Ti, np.eye(9), atol=1e-14)
    # A_n = T A_x T^-1 (rotational invariance of the elastic system)
    Aall = physics.jacobians(2500.0, 3e10, 2e10)
    An = np.einsum("d,dpq->pq", n, Aall)
    assert np.allclose(T @ Aall[0] @ Ti, An, atol=1e-9 * np.abs(An).max())


def test_flux_homogeneous_reduces_to_upwind_split():
    """Same material on both sides: A+- = (A_n +- |A_n|)/2 from an eigendecomposition."""
    rng = np.random.default_rng(4)
    n = rng.standard_normal(3); n /= np.linalg.norm(n)
    rho, vp = 2700.0, 5200.0
    lam, mu = physics.lame(rho, vp, vp / np.sqrt(3))
    Ap, Am = physics.flux_solvers(n, (rho, lam, mu), (rho, lam, mu))
    An = np.einsum("d,dpq->pq", n, physics.jacobians(rho, lam, mu))
    w, X = np.linalg.eig(An)
    absA = (X @ np.diag(np.abs(w)) @ np.linalg.inv(X)).real
    scale = np.abs(An).max()
    assert np.abs(Ap - 0.5 * (An + absA)).max() < 1e-9 * scale
    assert np.abs(Am - 0.5 * (An - absA)).max() < 1e-9 * scale


def test_flux_consistency_and_interface_conditions():
    """Heterogeneous: A+ + A- = A_n(m-); traction and velocity of q* agree from both sides."""
    rng = np.random.default_rng(5)
    n = rng.standard_normal(3); n /= np.linalg.norm(n)
    m1 = physics.lame(2100.0, 3300.0, 3300.0 / np.sqrt(3))
    m2 = physics.lame(2900.0, 5800.0, 5800.0 / np.sqrt(3))
    mat1 = (2100.0,) + m1
    mat2 = (2900.0,) + m2
    Ap, Am = physics.flux_solvers(n, mat1, mat2)
    An = np.einsum("d,dpq->pq", n, physics.jacobians(*mat1))
    assert np.abs(Ap + Am - An).max() < 1e-12 * np.abs(An).max()
    # Godunov states from both sides: traction sigma.n and velocity must coincide.
    q1 = rng.standard_normal(9) * np.r_[np.full(6, 1e6), np.ones(3)]
    q2 = rng.standard_normal(9) * np.r_[np.full(6, 1e6), np.ones(3)]

    def state(nrm, ma, mb, qa, qb):
        R = physics.face_frame(nrm)
        T, Ti = physics.rotation(R), physics.rotation(R.T)
        Zp = lambda m: np.sqrt(m[0] * (m[1] + 2 * m[2]))
        Zs = lambda m: np.sqrt(m[0] * m[2])
        Gm, Gp = physics.godunov_state(Zp(ma), Zs(ma), Zp(mb), Zs(mb))
        qs = T @ (Gm @ Ti @ qa + Gp @ Ti @ qb)
        S = np.array([[qs[0], qs[3], qs[5]], [qs[3], qs[1], qs[4]], [qs[5], qs[4], qs[2]]])
        return S @ nrm, qs[6:9]

    t1, v1 = state(n, mat1, mat2, q1, q2)
    t2, v2 = state(-n, mat2, mat1, q2, q1)
    assert np.allclose(t1, -t2, rtol=0, atol=1e-8 * np.abs(t1).max())  # t2 uses -n
    assert np.allclose(v1, v2, rtol=0, atol=1e-10 * max(1.0, np.abs(v1).max()))


def test_mesh_geometry_and_neighbours():
    cfg = synth.CONFIGS["c0"]
    xyz, vid = synth.kuhn_mesh(cfg.nx, cfg.ny, cfg.nz, seed=cfg.seed)
    J, Jinv, detJ, area, normal = mesh.geometry(xyz)
    assert (detJ > 0).all()
    # periodic jittered tiling: total volume equals the torus volume exactly (up to rounding)
    assert abs(detJ.sum() / 6.0 - cfg.nx * cfg.ny * cfg.nz) < 1e-10
    # closed surface: sum_i |S_i| n_i = 0 per element
    assert np.abs((area[..., None] * normal).sum(1)).max() < 1e-13
    nb, j, h = mesh.neighbour_table(vid)
    E = len(vid)
    e = np.arange(E)[:, None].repeat(4, 1)
    assert (nb[nb, j] == e).all()                       # Neigh(Neigh) = self, via Face
    # the shared face has opposite normals on the two sides
    assert np.abs(normal + normal[nb, j]).max() < 1e-12
    assert ((h >= 0) & (h <= 2)).all()


def test_face_matching_rejects_bad_mesh():
    xyz, vid = synth.kuhn_mesh(3, 3, 3)
    with pytest.raises(ValueError):
        mesh.match_faces(vid[:-1])
