"""Global matrices of the ADER-DG scheme by exact integration.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Definitions (reference element, orthonormal basis so M = I, reading R10):
  M_kl      = int_T phi_k phi_l                                   (mass)
  K^c_kl    = int_T (d phi_k / d xi_c) phi_l                      (P:323-332 stiffness)
  Ktilde^c  = -M^-1 (K^c)^T    derivative matrices of the CK recursion (R4)
  Khat^c    = +M^-1 K^c        volume matrices of the update           (R4)
  Fm^i_kl   = int_tri phi_k(x^(i)(chi,tau)) phi_l(x^(i)(chi,tau))  local face matrix
  Fp_kl     = int_tri phi_k(x^(i)(chi,tau)) phi_l(x_nb(chi,tau))    neighbour face matrix
  R^i_km    = int_tri phi_k(x^(i)(chi,tau)) psi_m(chi,tau)
  f^h_mn    = int_tri psi_m(chi,tau) psi_n(chit^h(chi,tau))

with the face parametrisations x^(i)(chi,tau) = P_a + chi (P_b - P_a) + tau (P_c - P_a)
for the outward-oriented vertex triples FACES (reading R7).  The step (``oracle.step``)
uses Fm and Fp only; R and f exist for the pins (Fm = R R^T, Fp = R^i f^h R^jT) and for the
literal einsum mode, which evaluates the paper's factored chain R f R I A- (P:1342).

Integrals are exact: polynomials with integer coefficients are multiplied against an
integer Gram matrix of monomial moments (scaled by a common factorial), and the
normalisation 1/sqrt(int phi~^2) is applied at the very end in 50-digit arithmetic,
then rounded once to fp64.
"""
from __future__ import annotations

from functools import lru_cache
from math import factorial

import mpmath
import numpy as np

from . import basis

# Reference tetrahedron vertices and the four outward-oriented face triples (reading R7).
REF_VERTS = ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1))
FACES = ((0, 2, 1), (0, 1, 3), (0, 3, 2), (1, 2, 3))

_DPS = 50


def _monomials3(D):
    return [(a, b, d - a - b) for d in range(D + 1) for a in range(d, -1, -1)
            for b in range(d - a, -1, -1)]


def _monomials2(D):
    return [(a, d - a) for d in range(D + 1) for a in range(d, -1, -1)]


def _coeff_matrix(polys, monos):
    idx = {m: i for i, m in enumerate(monos)}
    C = np.zeros((len(monos), len(polys)), dtype=object)
    C[:, :] = 0
    for k, p in enumerate(polys):
        for m, v in p.items():
            C[idx[m], k] = v
    return C


@lru_cache(maxsize=None)
def _gram3(N):
    """Integer Gram matrix G[a,b] = L * int_T m_a m_b of degree-<=N monomials, L=(2N+3)!."""
    monos = _monomials3(N)
    L = factorial(2 * N + 3)
    G = np.zeros((len(monos), len(monos)), dtype=object)
    for i, (a1, b1, c1) in enumerate(monos):
        for j, (a2, b2, c2) in enumerate(monos):
            a, b, c = a1 + a2, b1 + b2, c1 + c2
            G[i, j] = factorial(a) * factorial(b) * factorial(c) * (L // factorial(a + b + c + 3))
    return monos, G, L


@lru_cache(maxsize=None)
def _gram2(N):
    """Integer Gram matrix G[a,b] = L * int_tri m_a m_b, L=(2N+2)!."""
    monos = _monomials2(N)
    L = factorial(2 * N + 2)
    G = np.zeros((len(monos), len(monos)), dtype=object)
    for i, (a1, b1) in enumerate(monos):
        for j, (a2, b2) in enumerate(monos):
            a, b = a1 + a2, b1 + b2
            G[i, j] = factorial(a) * factorial(b) * (L // factorial(a + b + 2))
    return monos, G, L


def _to_float(raw_int, L, n2_row, n2_col):
    """raw_int / L / sqrt(n2_row[k] n2_col[l]) elementwise, rounded once to fp64."""
    out = np.zeros(raw_int.shape, dtype=np.float64)
    with mpmath.workdps(_DPS):
        sr = [mpmath.sqrt(mpmath.mpf(x.numerator) / x.denominator) for x in n2_row]
        sc = [mpmath.sqrt(mpmath.mpf(x.numerator) / x.denominator) for x in n2_col]
        for k in range(raw_int.shape[0]):
            for l in range(raw_int.shape[1]):
                v = raw_int[k, l]
                if v != 0:
                    out[k, l] = float(mpmath.mpf(v) / L / (sr[k] * sc[l]))
    return out


@lru_cache(maxsize=None)
def _tet_data(N):
    tb = basis.tet_basis(N)
    polys = [p for p, _ in tb]
    n2 = [n for _, n in tb]
    return polys, n2


@lru_cache(maxsize=None)
def _tri_data(N):
    tb = basis.tri_basis(N)
    return [p for p, _ in tb], [n for _, n in tb]


@lru_cache(maxsize=None)
def mass_matrix_exact(N):
    """Exact rational check data: (raw integer matrix, L, norms).  M = raw / L / sqrt(n n)."""
    polys, n2 = _tet_data(N)
    monos, G, L = _gram3(N)
    C = _coeff_matrix(polys, monos)
    raw = C.T.dot(G).dot(C)
    return raw, L, n2


def mass_matrix(N):
    raw, L, n2 = mass_matrix_exact(N)
    return _to_float(raw, L, n2, n2)


@lru_cache(maxsize=None)
def stiffness(N):
    """K^c_kl = int_T (d phi_k/d xi_c) phi_l, shape (3, B, B)."""
    polys, n2 = _tet_data(N)
    monos, G, L = _gram3(N)
    C = _coeff_matrix(polys, monos)
    GC = G.dot(C)
    K = []
    for c in range(3):
        Dc = _coeff_matrix([basis.p_deriv(p, c) for p in polys], monos)
        K.append(_to_float(Dc.T.dot(GC), L, n2, n2))
    return np.array(K)


def _mass_is_identity(N):
    raw, L, n2 = mass_matrix_exact(N)
    B = len(n2)
    for k in range(B):
        for l in range(B):
            want = n2[k] * L if k == l else 0
            if raw[k, l] != want:
                return False
    return True


@lru_cache(maxsize=None)
def derivative_matrices(N):
    """Ktilde^c = -M^-1 (K^c)^T  (reading R4).  M is exactly I (asserted in exact arithmetic)."""
    assert _mass_is_identity(N), "orthonormality of the basis failed in exact arithmetic"
    K = stiffness(N)
    return np.array([-K[c].T for c in range(3)])


@lru_cache(maxsize=None)
def volume_matrices(N):
    """Khat^c = M^-1 K^c  (reading R4)."""
    assert _mass_is_identity(N)
    return stiffness(N).copy()


def face_param(triple):
    """(origin, d1, d2) of x(chi,tau) = P_a + chi (P_b - P_a) + tau (P_c - P_a)."""
    a, b, c = (REF_VERTS[t] for t in triple)
    return a, tuple(bb - aa for aa, bb in zip(a, b)), tuple(cc - aa for aa, cc in zip(a, c))


@lru_cache(maxsize=None)
def _face_coeffs(N, triple):
    polys, n2 = _tet_data(N)
    o, d1, d2 = face_param(triple)
    restricted = [basis.restrict_to_face(p, o, d1, d2) for p in polys]
    monos, _, _ = _gram2(N)
    return _coeff_matrix(restricted, monos), n2


@lru_cache(maxsize=None)
def face_pair_matrix(N, triple_e, triple_nb):
    """int_tri phi_k(x_e(chi,tau)) phi_l(x_nb(chi,tau)) dchi dtau for two vertex triples.

    triple_e:  local vertex indices (a, b, c) of the face in the element,
    triple_nb: local vertex indices in the neighbour of the *same physical vertices*
               in the same order.  Fm^i = face_pair_matrix(N, FACES[i], FACES[i]).
    """
    Ce, n2 = _face_coeffs(N, tuple(triple_e))
    Cn, _ = _face_coeffs(N, tuple(triple_nb))
    _, G, L = _gram2(N)
    return _to_float(Ce.T.dot(G).dot(Cn), L, n2, n2)


def face_mass_matrix(N, i):
    """Fm^i (B x B)."""
    return face_pair_matrix(N, FACES[i], FACES[i])


@lru_cache(maxsize=None)
def lift_matrix(N, i):
    """R^i_km = int_tri phi_k(x^(i)) psi_m  (B x Btilde)."""
    Ce, n2 = _face_coeffs(N, FACES[i])
    tpolys, tn2 = _tri_data(N)
    monos, G, L = _gram2(N)
    Cpsi = _coeff_matrix(tpolys, monos)
    return _to_float(Ce.T.dot(G).dot(Cpsi), L, n2, tn2)


# chit^h(chi, tau) as (chi', tau') linear polynomials (reading R7).
_ROT = {
    0: ({(0, 1): 1}, {(1, 0): 1}),                                  # (tau, chi)
    1: ({(0, 0): 1, (1, 0): -1, (0, 1): -1}, {(0, 1): 1}),          # (1-chi-tau, tau)
    2: ({(1, 0): 1}, {(0, 0): 1, (1, 0): -1, (0, 1): -1}),          # (chi, 1-chi-tau)
}


def _compose2(poly2, chi_p, tau_p):
    out = {}
    for (a, b), v in poly2.items():
        term = basis.p_mul(basis.p_pow(chi_p, a, 2), basis.p_pow(tau_p, b, 2))
        out = basis.p_add(out, basis.p_scale(term, v))
    return out


@lru_cache(maxsize=None)
def rotation_matrix(N, h):
    """f^h_mn = int_tri psi_m(chi,tau) psi_n(chit^h(chi,tau))  (Btilde x Btilde)."""
    tpolys, tn2 = _tri_data(N)
    monos, G, L = _gram2(N)
    chi_p, tau_p = _ROT[h]
    Cpsi = _coeff_matrix(tpolys, monos)
    Crot = _coeff_matrix([_compose2(p, chi_p, tau_p) for p in tpolys], monos)
    return _to_float(Cpsi.T.dot(G).dot(Crot), L, tn2, tn2)


def basis_eval(N, pts):
    """phi_k at reference points pts (n,3), float64; used by pins (plane wave projection)."""
    polys, n2 = _tet_data(N)
    pts = np.asarray(pts, dtype=np.float64)
    out = np.zeros((pts.shape[0], len(polys)))
    for k, p in enumerate(polys):
        s = 1.0 / float(mpmath.sqrt(mpmath.mpf(n2[k].numerator) / n2[k].denominator))
        v = np.zeros(pts.shape[0])
        for (a, b, c), coef in p.items():
            v += float(coef) * pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c
        out[:, k] = v * s
    return out
