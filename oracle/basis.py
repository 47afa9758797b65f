"""Dubiner basis on the reference tetrahedron, face basis on the reference triangle.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The paper names the basis only as "Dubiner's basis functions" with
B = C(N+3,3) functions of maximum degree N and face matrices of size
B x Btilde, Btilde = C(N+2,2).  Reading R6 fixes the
formula, the ordering and the normalisation:

  reference tetrahedron T = {xi, eta, zeta >= 0, xi + eta + zeta <= 1},
  collapsed coordinates  a = 2 xi/(1-eta-zeta) - 1,  b = 2 eta/(1-zeta) - 1,  c = 2 zeta - 1,
  phi_pqr = P_p^(0,0)(a) ((1-b)/2)^p  P_q^(2p+1,0)(b) ((1-c)/2)^(p+q)  P_r^(2p+2q+2,0)(c),
  ordered by total degree d = p+q+r, then r, then q;  normalised to int_T phi^2 = 1.

Everything here is exact: each unnormalised phi is a polynomial with *integer*
coefficients in (xi, eta, zeta), obtained from the textbook Jacobi sum

  P_n^(al,be)(x) = sum_s C(n+al, n-s) C(n+be, s) ((x-1)/2)^s ((x+1)/2)^(n-s),

homogenised with the collapse factors: with (x-1)/2 = (X-W)/W and (x+1)/2 = X/W,
P_n^(al,0)(x) W^n = sum_s C(n+al, n-s) C(n, s) (X-W)^s X^(n-s).  The normalisation
constant is 1/sqrt(int phi~^2), kept as the exact rational int phi~^2.

Monomial integrals (exact):  int_T xi^a eta^b zeta^c = a! b! c! / (a+b+c+3)!,
                             int_tri chi^a tau^b     = a! b! / (a+b+2)!.
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache
from math import comb, factorial

# ---------------------------------------------------------------- polynomials
# A polynomial is a dict {exponent tuple: int coefficient}.


def p_add(p, q, s=1):
    r = dict(p)
    for k, v in q.items():
        r[k] = r.get(k, 0) + s * v
    return {k: v for k, v in r.items() if v != 0}


def p_mul(p, q):
    r = {}
    for k1, v1 in p.items():
        for k2, v2 in q.items():
            k = tuple(a + b for a, b in zip(k1, k2))
            r[k] = r.get(k, 0) + v1 * v2
    return {k: v for k, v in r.items() if v != 0}


def p_pow(p, n, nvar):
    r = {(0,) * nvar: 1}
    for _ in range(n):
        r = p_mul(r, p)
    return r


def p_scale(p, s):
    return {k: v * s for k, v in p.items() if v * s != 0}


def p_deriv(p, var):
    """Partial derivative with respect to variable index ``var``."""
    r = {}
    for k, v in p.items():
        if k[var] > 0:
            kk = list(k)
            kk[var] -= 1
            r[tuple(kk)] = r.get(tuple(kk), 0) + v * k[var]
    return {k: v for k, v in r.items() if v != 0}


def p_eval(p, x):
    """Evaluate at a point (floats or Fractions)."""
    tot = 0
    for k, v in p.items():
        t = v
        for xi, e in zip(x, k):
            t = t * xi ** e
        tot += t
    return tot


def jacobi_homogenised(n, alpha, X, W, nvar):
    """P_n^(alpha,0)(x) * W^n with (x+1)/2 = X/W, as an integer polynomial (X, W polys)."""
    out = {}
    XmW = p_add(X, W, -1)
    for s in range(n + 1):
        c = comb(n + alpha, n - s) * comb(n, s)
        term = p_mul(p_pow(XmW, s, nvar), p_pow(X, n - s, nvar))
        out = p_add(out, p_scale(term, c))
    return out


# ------------------------------------------------------------- tetrahedron


def n_basis(N):
    """B = C(N+3, 3)."""
    return comb(N + 3, 3)


def n_face_basis(N):
    """Btilde = C(N+2, 2)."""
    return comb(N + 2, 2)


def tet_index(N):
    """List of (p, q, r) in the basis order of reading R6: degree, then r, then q."""
    out = []
    for d in range(N + 1):
        for r in range(d + 1):
            for q in range(d - r + 1):
                out.append((d - q - r, q, r))
    return out


_XI = {(1, 0, 0): 1}
_ETA = {(0, 1, 0): 1}
_ZETA = {(0, 0, 1): 1}
_ONE3 = {(0, 0, 0): 1}


@lru_cache(maxsize=None)
def tet_phi_unnormalised(p, q, r):
    """phi~_pqr as an integer polynomial in (xi, eta, zeta)."""
    w1 = p_add(p_add(_ONE3, _ETA, -1), _ZETA, -1)  # 1 - eta - zeta
    w2 = p_add(_ONE3, _ZETA, -1)  # 1 - zeta
    f1 = jacobi_homogenised(p, 0, _XI, w1, 3)  # P_p(a) ((1-b)/2)^p (1-zeta)^p
    f2 = jacobi_homogenised(q, 2 * p + 1, _ETA, w2, 3)  # P_q(b) (1-zeta)^q
    f3 = jacobi_homogenised(r, 2 * p + 2 * q + 2, _ZETA, _ONE3, 3)  # P_r(c)
    return p_mul(p_mul(f1, f2), f3)


def tet_monomial_integral(a, b, c):
    return Fraction(factorial(a) * factorial(b) * factorial(c), factorial(a + b + c + 3))


def tet_integral(p):
    return sum((v * tet_monomial_integral(*k) for k, v in p.items()), Fraction(0))


@lru_cache(maxsize=None)
def tet_norm2(p, q, r):
    """int_T phi~_pqr^2, exact."""
    f = tet_phi_unnormalised(p, q, r)
    return tet_integral(p_mul(f, f))


def tet_basis(N):
    """[(phi~_k integer polynomial, int_T phi~_k^2 exact), ...] in basis order."""
    return [(tet_phi_unnormalised(*t), tet_norm2(*t)) for t in tet_index(N)]


# ---------------------------------------------------------------- triangle

_CHI = {(1, 0): 1}
_TAU = {(0, 1): 1}
_ONE2 = {(0, 0): 1}


def tri_index(N):
    """List of (p, q) for the face basis: degree, then q."""
    out = []
    for d in range(N + 1):
        for q in range(d + 1):
            out.append((d - q, q))
    return out


@lru_cache(maxsize=None)
def tri_psi_unnormalised(p, q):
    """psi~_pq(chi, tau) = P_p(2chi/(1-tau) - 1)(1-tau)^p P_q^(2p+1,0)(2tau - 1)."""
    w = p_add(_ONE2, _TAU, -1)
    f1 = jacobi_homogenised(p, 0, _CHI, w, 2)
    f2 = jacobi_homogenised(q, 2 * p + 1, _TAU, _ONE2, 2)
    return p_mul(f1, f2)


def tri_monomial_integral(a, b):
    return Fraction(factorial(a) * factorial(b), factorial(a + b + 2))


def tri_integral(p):
    return sum((v * tri_monomial_integral(*k) for k, v in p.items()), Fraction(0))


@lru_cache(maxsize=None)
def tri_norm2(p, q):
    f = tri_psi_unnormalised(p, q)
    return tri_integral(p_mul(f, f))


def tri_basis(N):
    return [(tri_psi_unnormalised(*t), tri_norm2(*t)) for t in tri_index(N)]


# ------------------------------------------------------- affine restriction


def restrict_to_face(poly3, origin, d1, d2):
    """poly3(origin + chi*d1 + tau*d2) as an integer polynomial in (chi, tau).

    origin, d1, d2 are integer 3-vectors (the reference tetrahedron's vertices are
    0/1 points, so every face parametrisation used here is integral).
    """
    lin = []
    for ax in range(3):
        f = {}
        if origin[ax]:
            f[(0, 0)] = origin[ax]
        if d1[ax]:
            f[(1, 0)] = d1[ax]
        if d2[ax]:
            f[(0, 1)] = d2[ax]
        lin.append(f)
    powcache = {}

    def lp(ax, e):
        key = (ax, e)
        if key not in powcache:
            powcache[key] = p_pow(lin[ax], e, 2)
        return powcache[key]

    out = {}
    for (a, b, c), v in poly3.items():
        term = p_mul(p_mul(lp(0, a), lp(1, b)), lp(2, c))
        out = p_add(out, p_scale(term, v))
    return out
