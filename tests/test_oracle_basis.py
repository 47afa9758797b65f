"""Pins of the oracle's basis and global matrices (oracle/basis.py, oracle/matrices.py).

Each pin is something other than the oracle's own formula: exact rational identities,
an independent scipy Gauss-Jacobi quadrature with scipy Jacobi polynomials, closed-form
derivatives of monomials, and the structural facts the paper states.
"""
from math import comb, factorial, sqrt

import numpy as np
import pytest

from oracle import basis, matrices
from tests import quadrature as qd

NS = [1, 2, 3, 4, 5, 6]


@pytest.mark.parametrize("N", NS)
def test_mass_matrix_is_exact_identity(N):
    # orthonormality in exact rational arithmetic (reading R10: M = I)
    assert matrices._mass_is_identity(N)
    assert np.array_equal(matrices.mass_matrix(N), np.eye(comb(N + 3, 3)))


def test_sizes():
    for N in NS:
        assert len(basis.tet_index(N)) == comb(N + 3, 3)   # B
        assert len(basis.tri_index(N)) == comb(N + 2, 2)   # Btilde


@pytest.mark.parametrize("N", [2, 5])
def test_basis_matches_scipy_jacobi(N):
    """Oracle polynomial expansion == scipy Jacobi evaluation in collapsed coordinates."""
    pts, w = qd.tet_rule(N + 2)
    ref = qd.dubiner_scipy(N, pts)
    norms = np.sqrt((ref ** 2 * w[:, None]).sum(0))
    ref = ref / norms
    got = matrices.basis_eval(N, pts)
    assert np.abs(got - ref).max() < 1e-11
    # independent quadrature also sees an orthonormal basis
    M = (got * w[:, None]).T @ got
    assert np.abs(M - np.eye(M.shape[0])).max() < 1e-12


def test_phi0_and_zero_means():
    N = 4
    pts, w = qd.tet_rule(N + 2)
    phi = matrices.basis_eval(N, pts)
    assert np.allclose(phi[:, 0], sqrt(6.0), atol=1e-14, rtol=0)  # |T| = 1/6
    means = (phi * w[:, None]).sum(0)
    assert abs(means[0] - sqrt(6.0) / 6) < 1e-14
    assert np.abs(means[1:]).max() < 1e-13


@pytest.mark.parametrize("N", [3, 5])
def test_hierarchical_span(N):
    """The first C(n+3,3) functions span all monomials of degree <= n (exact check)."""
    polys = [p for p, _ in basis.tet_basis(N)]
    for n in range(N + 1):
        Bn = comb(n + 3, 3)
        for f in polys[:Bn]:
            assert max(sum(k) for k in f) <= n
        monos = sorted({k for f in polys[:Bn] for k in f})
        assert len(monos) == Bn
        C = np.array([[float(f.get(m, 0)) for m in monos] for f in polys[:Bn]])
        assert np.linalg.matrix_rank(C) == Bn


def _mono_val(pts, a, b, c):
    return pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c


@pytest.mark.parametrize("N", [2, 4, 6])
def test_derivative_matrix_differentiates_exactly(N):
    """Ktilde^c coeffs(p) = -coeffs(d_c p) for every monomial p of degree <= N (closed form)."""
    pts, w = qd.tet_rule(N + 2)
    phi = matrices.basis_eval(N, pts)
    Kt = matrices.derivative_matrices(N)
    for d in range(N + 1):
        for a in range(d + 1):
            for b in range(d - a + 1):
                c = d - a - b
                coeff = (phi * (w * _mono_val(pts, a, b, c))[:, None]).sum(0)
                exps = (a, b, c)
                for ax in range(3):
                    e = list(exps)
                    if e[ax] == 0:
                        deriv = np.zeros(len(w))
                    else:
                        k = e[ax]
                        e[ax] -= 1
                        deriv = k * _mono_val(pts, *e)
                    dcoeff = (phi * (w * deriv)[:, None]).sum(0)
                    assert np.abs(Kt[ax] @ coeff + dcoeff).max() < 2e-11


@pytest.mark.parametrize("N", NS)
def test_staircase_and_zero_blocks(N):
    """pattern(Ktilde) = pattern(Khat^T), D^d has C(N-d+3,3) nonzero rows;
    reading R3: Khat has exactly C(N+2,3) nonzero columns (not Btilde, garbled P:1352)."""
    Kt = matrices.derivative_matrices(N)
    Kh = matrices.volume_matrices(N)
    for c in range(3):
        assert np.array_equal(Kt[c] != 0, Kh[c].T != 0)
    for d in range(N + 1):
        rows_in = comb(N - d + 3, 3)
        rows_out = comb(N - d - 1 + 3, 3) if d < N else 0
        for c in range(3):
            blk = Kt[c][:, :rows_in]
            assert not blk[rows_out:].any()
    ncol = comb(N + 2, 3)
    nonzero_cols = np.any(np.stack([Kh[c] != 0 for c in range(3)]), axis=(0, 1))
    assert nonzero_cols[:ncol].all() and not nonzero_cols[ncol:].any()


def test_derivative_recursion_terminates():
    """Applying Ktilde N+1 times to anything gives exactly 0 (degree drops by one each time)."""
    N = 5
    Kt = matrices.derivative_matrices(N)
    rng = np.random.default_rng(0)
    v = rng.standard_normal(comb(N + 3, 3))
    for c_seq in [(0,) * (N + 1), (2, 1, 0, 2, 1, 0)]:
        x = v.copy()
        for c in c_seq[: N + 1]:
            x = Kt[c] @ x
        assert np.abs(x).max() == 0.0


@pytest.mark.parametrize("N", [2, 5])
def test_face_matrices_quadrature_and_factorisation(N):
    """Fm^i by independent triangle quadrature; Fm^i = R^i R^iT; f^h orthogonal; and the
    paper's factorisation R^i f^h R^jT equals the directly integrated neighbour matrix."""
    tpts, tw = qd.tri_rule(N + 2)
    for i, tri in enumerate(matrices.FACES):
        o, d1, d2 = (np.array(v, dtype=float) for v in matrices.face_param(tri))
        x = o[None] + tpts[:, :1] * d1[None] + tpts[:, 1:] * d2[None]
        phi = matrices.basis_eval(N, x)
        Fq = (phi * tw[:, None]).T @ phi
        Fm = matrices.face_mass_matrix(N, i)
        assert np.abs(Fq - Fm).max() < 1e-12 * np.abs(Fm).max()  # monomial evaluation rounding
        R = matrices.lift_matrix(N, i)
        assert np.abs(R @ R.T - Fm).max() < 1e-12
    for h in range(3):
        f = matrices.rotation_matrix(N, h)
        assert np.abs(f @ f.T - np.eye(f.shape[0])).max() < 1e-13
    # R f R^T for every (i, j, h) vs direct integration with the vertex correspondence
    faces = matrices.FACES
    for i in range(4):
        for j in range(4):
            for h in range(3):
                # neighbour triple is a rotation of the reversed triple (reading R7)
                a, b, c = "a", "b", "c"
                rev = [a, c, b]
                rot = rev[-h:] + rev[:-h] if h else rev
                assert rot.index(a) == h
                # local vertices of the neighbour carrying the element's (a, b, c)
                nb_local = {lab: faces[j][pos] for pos, lab in enumerate(rot)}
                triple_nb = (nb_local["a"], nb_local["b"], nb_local["c"])
                Fp = matrices.face_pair_matrix(N, faces[i], triple_nb)
                Rf = matrices.lift_matrix(N, i) @ matrices.rotation_matrix(N, h) @ matrices.lift_matrix(N, j).T
                assert np.abs(Fp - Rf).max() < 1e-12


def test_divergence_theorem_on_reference():
    """int_T d_c phi_k = sum_i int_{S_i} phi_k n_ic dS links K^c (volume) to Fm (faces)."""
    N = 4
    K = matrices.stiffness(N)
    ref = np.array(matrices.REF_VERTS, dtype=float)
    lhs = K[:, :, 0] / sqrt(6.0)  # int d_c phi_k = K^c_k0 / phi_0
    rhs = np.zeros_like(lhs)
    for i, (a, b, c) in enumerate(matrices.FACES):
        cr = np.cross(ref[b] - ref[a], ref[c] - ref[a])  # = 2|S| n
        Fm = matrices.face_mass_matrix(N, i)
        int_phi = Fm[:, 0] / sqrt(6.0)  # int_tri phi_k dchi dtau
        rhs += cr[:, None] * int_phi[None, :]
    assert np.abs(lhs - rhs).max() < 1e-13


def test_monomial_integrals_closed_form():
    # int_T 1 = 1/6, int_T xi = 1/24, int_tri 1 = 1/2 (textbook values)
    from fractions import Fraction
    assert basis.tet_monomial_integral(0, 0, 0) == Fraction(1, 6)
    assert basis.tet_monomial_integral(1, 0, 0) == Fraction(1, 24)
    assert basis.tri_monomial_integral(0, 0) == Fraction(1, 2)
    assert basis.tet_monomial_integral(2, 1, 1) == Fraction(2 * 1 * 1, factorial(7))
