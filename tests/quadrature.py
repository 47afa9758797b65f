"""Independent numerical quadrature used by the oracle pins (not by the oracle itself).

Stroud conical-product rule on the reference tetrahedron from scipy's Gauss-Jacobi roots,
and the Dubiner functions evaluated directly from scipy's Jacobi polynomials in collapsed
coordinates -- a second, numerical construction to pin the oracle's exact rational one.
"""
import numpy as np
from scipy.special import eval_jacobi, roots_jacobi


def tet_rule(n):
    """Points (m,3) and weights (m,) exact for polynomials of degree <= 2n-1 on T."""
    a, wa = roots_jacobi(n, 0, 0)
    b, wb = roots_jacobi(n, 1, 0)
    c, wc = roots_jacobi(n, 2, 0)
    A, Bq, C = np.meshgrid(a, b, c, indexing="ij")
    W = (wa[:, None, None] * wb[None, :, None] * wc[None, None, :]) / 64.0
    xi = (1 + A) * (1 - Bq) * (1 - C) / 8.0
    eta = (1 + Bq) * (1 - C) / 4.0
    zeta = (1 + C) / 2.0
    return np.stack([xi.ravel(), eta.ravel(), zeta.ravel()], axis=1), W.ravel()


def tri_rule(n):
    """Points (m,2), weights on {chi,tau >= 0, chi+tau <= 1}, exact to degree 2n-1."""
    a, wa = roots_jacobi(n, 0, 0)
    b, wb = roots_jacobi(n, 1, 0)
    A, Bq = np.meshgrid(a, b, indexing="ij")
    W = (wa[:, None] * wb[None, :]) / 8.0
    chi = (1 + A) * (1 - Bq) / 4.0
    tau = (1 + Bq) / 2.0
    return np.stack([chi.ravel(), tau.ravel()], axis=1), W.ravel()


def dubiner_scipy(N, pts):
    """Unnormalised phi_pqr at points, ordered by degree, then r, then q (reading R6)."""
    xi, eta, zeta = pts[:, 0], pts[:, 1], pts[:, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        a = np.where(np.abs(1 - eta - zeta) > 1e-300, 2 * xi / (1 - eta - zeta) - 1, -1.0)
        b = np.where(np.abs(1 - zeta) > 1e-300, 2 * eta / (1 - zeta) - 1, -1.0)
    c = 2 * zeta - 1
    cols = []
    for d in range(N + 1):
        for r in range(d + 1):
            for q in range(d - r + 1):
                p = d - q - r
                v = (eval_jacobi(p, 0, 0, a) * ((1 - b) / 2) ** p * eval_jacobi(q, 2 * p + 1, 0, b)
                     * ((1 - c) / 2) ** (p + q) * eval_jacobi(r, 2 * p + 2 * q + 2, 0, c))
                cols.append(v)
    return np.stack(cols, axis=1)
