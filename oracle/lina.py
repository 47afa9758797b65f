"""LinA: ADER-DG-SEM for the linearised acoustic equations on uniform cuboid grids (3D).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Row NEXT-3 of SURVEY §8(f).

The paper's scheme (§"LinA"), with a tensor-product nodal basis
q_p = Q_lmnp psi_l(x) psi_m(y) psi_n(z):

  D^(d+1)_xyzp = Kt_xl D^d_lyzq A*_pq + Kt_ym D^d_xmzq B*_pq + Kt_zn D^d_xynq C*_pq,  D^0 = Q
  I_xyzp       = sum_{d=0}^{N} dt^(d+1)/(d+1)! D^d_xyzp
  Q*_xyzp      = Q_xyzp + Kh_xl I_lyzq A*_pq + Kh_ym I_xmzq B*_pq + Kh_zn I_xynq C*_pq
  X^s_yzp = F^s_l I_lyzp,  Y^s_xzp = F^s_m I_xmzp,  Z^s_xyp = F^s_n I_xynp,  F^left_i = d_i0,
  F^right_i = d_iN
  Q^(n+1)_xyzp = Q*_xyzp + sum_{s in left,right} Fh^s_x (X^s_yzq (A+)^s_pq + X^Neigh(s)_yzq (A-)^s_pq)
                 + (the same along y with Y, along z with Z)

Readings (L1-L8) where the paper is silent:
L1  quantities q = (p, u, v, w); p_t + K (u_x + v_y + w_z) = 0, rho v_t + grad p = 0
    (linearised acoustics, LeVeque 2002, cited at P:1455), written q_t + A q_x + B q_y + C q_z = 0;
    per-element bulk modulus K and density rho.
L2  1D basis: Lagrange polynomials psi_i on the N+1 Gauss-Lobatto-Legendre points of [0, 1]
    ("nodal basis with Gauss-Lobatto points"), so Q is the nodal values.
L3  DG-SEM collocation (Kopriva 2009 ch. 5.4, cited at P:1461): the mass matrix is the GLL
    quadrature diag(w) (lumped); the stiffness integrals int psi'_k psi_l (degree 2N-1) are exact.
L4  Kt = -Dm with Dm_kl = psi'_l(xi_k) (the nodal derivative), A* = A / h_x, B* = B / h_y,
    C* = C / h_z: D^(d+1) = -(A d_x + B d_y + C d_z) D^d exactly for the nodal interpolant.
L5  Kh_kl = (1 / w_k) int_0^1 psi'_k psi_l = w_l Dm_lk / w_k (weak-form volume term).
L6  Fh^left_x = -d_x0 / w_0, Fh^right_x = -d_xN / w_N: the boundary term -psi_k F*_n of the
    weak form with the OUTWARD normal flux F*_n, scaled by the lumped mass; (A+-)^s =
    A^(+-)_n / h with n the outward normal of side s (so both ends carry the same sign).
L7  numerical flux: exact Godunov state of the 1D acoustic interface problem with both
    materials, F* = A_n(m-) q*:  with Z = sqrt(rho K), normal velocity u_n = n . v,
      p*   = (Z+ p- + Z- p+ + Z- Z+ (u_n- - u_n+)) / (Z- + Z+),
      u_n* = (Z- u_n- + Z+ u_n+ + p- - p+) / (Z- + Z+),
      A_n q* = (K- u_n*, p* n / rho-),  so A+ q- + A- q+ = A_n(m-) q*.
L8  grid: nx x ny x nz periodic cuboids of size hx x hy x hz, element e = i + nx (j + ny k);
    Neigh(left/right) = (i -+ 1 mod nx, j, k) etc.; the neighbour's trace on the shared
    face is its opposite side (right <-> left).
Arrays: Q[e, x, y, z, p] (element, then the node indices along x, y, z, then quantity).
"""
from __future__ import annotations

from dataclasses import dataclass
from math import factorial

import mpmath
import numpy as np

mpmath.mp.dps = 40
SIDES = ((0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1))  # (axis, 0 = left/bottom/back, 1 = right/top/front)


def gll(N):
    """(nodes, weights) of the N+1-point Gauss-Lobatto-Legendre rule on [0, 1] (40 digits,
    rounded once): endpoints and the roots of P_N'; w_i = 1 / (N (N+1) P_N(x_i)^2) on [0,1]."""
    xs = [mpmath.mpf(-1)]
    dP = lambda x: mpmath.diff(lambda t: mpmath.legendre(N, t), x)
    # interior GLL points: roots of P_N' (numpy's fp64 roots, polished by Newton in 40 digits)
    for r in sorted(np.polynomial.legendre.Legendre.basis(N).deriv().roots().real):
        xs.append(mpmath.findroot(dP, mpmath.mpf(float(r))))
    xs.append(mpmath.mpf(1))
    xs = sorted(xs)
    ws = [mpmath.mpf(2) / (N * (N + 1) * mpmath.legendre(N, x) ** 2) for x in xs]
    return [(x + 1) / 2 for x in xs], [w / 2 for w in ws]


def derivative_matrix(nodes):
    """Dm_kl = psi'_l(xi_k) of the Lagrange basis on `nodes` (barycentric formula, mpmath)."""
    n = len(nodes)
    lam = [1 / mpmath.fprod([nodes[j] - nodes[m] for m in range(n) if m != j]) for j in range(n)]
    D = [[mpmath.mpf(0)] * n for _ in range(n)]
    for k in range(n):
        for l in range(n):
            if k != l:
                D[k][l] = (lam[l] / lam[k]) / (nodes[k] - nodes[l])
        D[k][k] = -mpmath.fsum(D[k][l] for l in range(n) if l != k)
    return D


def matrices(N):
    """(nodes, w, Kt, Kh, Fhat) in fp64: Kt = -Dm (L4), Kh = W^-1 Dm^T W (L5), Fhat[side end]
    (L6) as length-(N+1) vectors for end 0 (left) and 1 (right)."""
    nodes, w = gll(N)
    D = derivative_matrix(nodes)
    n = N + 1
    Kt = np.array([[float(-D[k][l]) for l in range(n)] for k in range(n)])
    Kh = np.array([[float(w[l] * D[l][k] / w[k]) for l in range(n)] for k in range(n)])
    Fh = np.zeros((2, n))
    Fh[0, 0] = float(-1 / w[0])
    Fh[1, N] = float(-1 / w[N])
    return np.array([float(x) for x in nodes]), np.array([float(x) for x in w]), Kt, Kh, Fh


def jacobians(rho, K):
    """A, B, C (L1) for q = (p, u, v, w)."""
    J = np.zeros((3, 4, 4))
    for a in range(3):
        J[a, 0, 1 + a] = K
        J[a, 1 + a, 0] = 1.0 / rho
    return J


def flux_solvers(axis, sign, m_own, m_nb):
    """(A+, A-) of L7 for the outward normal n = sign e_axis: A+ q- + A- q+ = A_n(m-) q*."""
    rho_m, K_m = m_own
    rho_p, K_p = m_nb
    Zm, Zp = np.sqrt(rho_m * K_m), np.sqrt(rho_p * K_p)
    S = Zm + Zp
    n = np.zeros(3)
    n[axis] = sign
    # (p*, u_n*) = G- q- + G+ q+
    Gm = np.zeros((2, 4))
    Gp = np.zeros((2, 4))
    Gm[0, 0] = Zp / S
    Gm[0, 1:] = Zm * Zp / S * n
    Gp[0, 0] = Zm / S
    Gp[0, 1:] = -Zm * Zp / S * n
    Gm[1, 0] = 1.0 / S
    Gm[1, 1:] = Zm / S * n
    Gp[1, 0] = -1.0 / S
    Gp[1, 1:] = Zp / S * n
    # F = (K- u_n*, p* n / rho-)
    T = np.zeros((4, 2))
    T[0, 1] = K_m
    T[1:, 0] = n / rho_m
    return T @ Gm, T @ Gp


@dataclass
class Grid:
    N: int
    nx: int
    ny: int
    nz: int
    h: tuple          # (hx, hy, hz)
    Kt: np.ndarray
    Kh: np.ndarray
    Fh: np.ndarray    # (2, N+1)
    w: np.ndarray
    nodes: np.ndarray
    Astar: np.ndarray  # (E, 3, 4, 4)
    Aplus: np.ndarray  # (E, 6, 4, 4) with the 1/h of the side's axis folded in
    Aminus: np.ndarray
    nb: np.ndarray     # (E, 6)

    @property
    def E(self):
        return self.nx * self.ny * self.nz


def neighbours(nx, ny, nz):
    """nb[e, side] of the periodic grid (L8), sides in SIDES order."""
    E = nx * ny * nz
    e = np.arange(E)
    i, j, k = e % nx, (e // nx) % ny, e // (nx * ny)
    idx = lambda a, b, c: (a % nx) + nx * ((b % ny) + ny * (c % nz))
    return np.stack([idx(i - 1, j, k), idx(i + 1, j, k), idx(i, j - 1, k), idx(i, j + 1, k),
                     idx(i, j, k - 1), idx(i, j, k + 1)], axis=1)


def setup(N, nx, ny, nz, h, material):
    """material: (E, 2) = (rho, K) per element."""
    nodes, w, Kt, Kh, Fh = matrices(N)
    E = nx * ny * nz
    nb = neighbours(nx, ny, nz)
    Astar = np.zeros((E, 3, 4, 4))
    Ap = np.zeros((E, 6, 4, 4))
    Am = np.zeros((E, 6, 4, 4))
    for e in range(E):
        J = jacobians(*material[e])
        for a in range(3):
            Astar[e, a] = J[a] / h[a]
        for s, (a, end) in enumerate(SIDES):
            p, m = flux_solvers(a, 1.0 if end else -1.0, material[e], material[nb[e, s]])
            Ap[e, s] = p / h[a]
            Am[e, s] = m / h[a]
    return Grid(N, nx, ny, nz, tuple(h), Kt, Kh, Fh, w, nodes, Astar, Ap, Am, nb)


def _apply3(M, T, Astar):
    """M_xl T_lyzq A*_pq + M_ym T_xmzq B*_pq + M_zn T_xynq C*_pq for T (E, n, n, n, 4)."""
    return (np.einsum("xl,elyzq,epq->exyzp", M, T, Astar[:, 0])
            + np.einsum("ym,exmzq,epq->exyzp", M, T, Astar[:, 1])
            + np.einsum("zn,exynq,epq->exyzp", M, T, Astar[:, 2]))


def time_integral(g: Grid, Q, dt):
    """(I, [D^0..D^N]) of P:1491-1499."""
    D = Q.copy()
    Ds = [D]
    I = dt * D
    for d in range(g.N):
        D = _apply3(g.Kt, D, g.Astar)
        Ds.append(D)
        I = I + dt ** (d + 2) / factorial(d + 2) * D
    return I, Ds


def sides(g: Grid, I):
    """X^s, Y^s, Z^s of P:1517-1521 for every side s (SIDES order): (E, 6, n, n, 4)."""
    n = g.N + 1
    F = np.zeros((2, n))
    F[0, 0] = 1.0
    F[1, g.N] = 1.0
    out = np.zeros((I.shape[0], 6, n, n, 4))
    for s, (a, end) in enumerate(SIDES):
        spec = ("l,elyzp->eyzp", "m,exmzp->exzp", "n,exynp->exyp")[a]
        out[:, s] = np.einsum(spec, F[end], I)
    return out


def update(g: Grid, Q, I):
    """Q^(n+1) of P:1506-1536 (volume, then the six sides' local and neighbour fluxes)."""
    out = Q + _apply3(g.Kh, I, g.Astar)
    X = sides(g, I)
    opposite = (1, 0, 3, 2, 5, 4)
    for s, (a, end) in enumerate(SIDES):
        own = X[:, s]
        nbt = X[g.nb[:, s], opposite[s]]
        flux = np.einsum("eabq,epq->eabp", own, g.Aplus[:, s]) + np.einsum("eabq,epq->eabp", nbt, g.Aminus[:, s])
        spec = ("x,eyzp->exyzp", "y,exzp->exyzp", "z,exyp->exyzp")[a]
        out = out + np.einsum(spec, g.Fh[end], flux)
    return out


def step(g: Grid, Q, dt, nsteps=1):
    for _ in range(nsteps):
        I, _ = time_integral(g, Q, dt)
        Q = update(g, Q, I)
    return Q
