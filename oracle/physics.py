"""Physics of the elastic / viscoelastic wave equation: Jacobians, star matrices, flux solvers.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The paper states only the generic linear system  dq/dt + A dq/dx + B dq/dy + C dq/dz = 0
(P:290-296), that the star matrices are "element-dependent linear combinations of the
Jacobians" and that A+, A- "contain the solution to the 1D Riemann problem"
(P:1348-1349).  Readings:

R5  velocity-stress elasticity, quantity order (sxx, syy, szz, sxy, syz, sxz, u, v, w):
      d_t sigma_ij = lam delta_ij div v + mu (d_i v_j + d_j v_i),   rho d_t v_i = sum_j d_j sigma_ij
    written as d_t q + sum_d A^d d_d q = 0 (the Jacobians are built from these continuum
    equations, not from a typed table; the test pins them against the table).
    Star matrices  A*^c = sum_d (J^-1)_cd A^d.
R8  exact Godunov (upwind) interface state for the face-normal 1D problem with both
    materials; flux F* = T Ahat(m-) q*,  q* = G- T^-1 q- + G+ T^-1 q+, so
    A+ = T Ahat(m-) G- T^-1 and A- = T Ahat(m-) G+ T^-1 (Ahat = x-Jacobian in the face frame).
R14 viscoelastic memory-variable form with 3 mechanisms (P = 27; quantities 9..26 are
    theta^l_(xx,yy,zz,xy,yz,xz), l = 0,1,2):
      d_t sigma - C_u : eps(v) = - sum_l Y_l : theta^l,   (Y:th)_ij = Ylam tr(th) delta_ij + 2 Ymu th_ij
      rho d_t v - div sigma = 0
      d_t theta^l - omega_l eps(v) = - omega_l theta^l,   eps = sym grad v (tensor strain rate)
    i.e. d_t q + sum_d A^d d_d q = E q.  The Riemann state is the elastic one (unrelaxed
    moduli); memory-variable rows of A+- follow from v*.  Parity only: physically unpinned.
"""
from __future__ import annotations

import numpy as np

# Voigt order of symmetric tensors: xx, yy, zz, xy, yz, xz
VOIGT = ((0, 0), (1, 1), (2, 2), (0, 1), (1, 2), (0, 2))
N_ELASTIC = 9
N_MECH = 3


def _voigt_index(i, j):
    for v, (a, b) in enumerate(VOIGT):
        if (a, b) == (i, j) or (a, b) == (j, i):
            return v
    raise KeyError


def lame(rho, vp, vs):
    """(lam, mu) from density and wave speeds."""
    mu = rho * vs * vs
    lam = rho * vp * vp - 2.0 * mu
    return lam, mu


def jacobians(rho, lam, mu, P=9, omega=None):
    """A^d (d = x, y, z), each P x P, for  d_t q + sum_d A^d d_d q = E q  (reading R5 / R14)."""
    A = np.zeros((3, P, P))
    delta = np.eye(3)
    for d in range(3):
        # stress rows: -(lam delta_ij delta_kd + mu (delta_id delta_jk + delta_jd delta_ik)) on v_k
        for s, (i, j) in enumerate(VOIGT):
            for k in range(3):
                coef = lam * delta[i, j] * delta[k, d] + mu * (delta[i, d] * delta[j, k] + delta[j, d] * delta[i, k])
                A[d, s, 6 + k] = -coef
        # velocity rows: rho d_t v_i = sum_m d_m sigma_im
        for i in range(3):
            for m in range(3):
                if m == d:
                    A[d, 6 + i, _voigt_index(i, m)] += -1.0 / rho
        # memory variables: d_t theta_ij - omega eps_ij = ..., eps_ij = (d_i v_j + d_j v_i)/2
        if P == 27:
            for l in range(N_MECH):
                for s, (i, j) in enumerate(VOIGT):
                    for k in range(3):
                        coef = 0.5 * (delta[i, d] * delta[j, k] + delta[j, d] * delta[i, k])
                        if coef != 0.0:
                            A[d, 9 + 6 * l + s, 6 + k] = -omega[l] * coef
    return A


def source_matrix(omega, Ylam, Ymu):
    """E (27 x 27) of reading R14: d_t q + ... = E q.  Ylam, Ymu: arrays of 3."""
    E = np.zeros((27, 27))
    for l in range(N_MECH):
        for s, (i, j) in enumerate(VOIGT):
            # (Y:theta)_ij = Ylam tr(theta) delta_ij + 2 Ymu theta_ij  enters d_t sigma with a minus
            for t, (a, b) in enumerate(VOIGT):
                coef = 0.0
                if i == j and a == b:
                    coef += Ylam[l]
                if s == t:
                    coef += 2.0 * Ymu[l]
                if coef != 0.0:
                    E[s, 9 + 6 * l + t] = -coef
            E[9 + 6 * l + s, 9 + 6 * l + s] = -omega[l]
    return E


def star_matrices(Jinv, A):
    """A*^c = sum_d (J^-1)_cd A^d."""
    return np.einsum("cd,dpq->cpq", Jinv, A)


def face_frame(n):
    """Orthonormal (n, s, t) with n the given unit normal; returned as columns of R."""
    n = np.asarray(n, dtype=np.float64)
    a = np.array([1.0, 0.0, 0.0]) if abs(n[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    s = a - n * np.dot(a, n)
    s /= np.linalg.norm(s)
    t = np.cross(n, s)
    return np.stack([n, s, t], axis=1)


def rotation(R, P=9):
    """T with q_global = T q_face for the frame R (columns n, s, t).

    Symmetric tensors rotate as S_g = R S_f R^T, vectors as v_g = R v_f.  Built by applying
    the rotation to each unit quantity vector (no closed-form Bond matrix typed in).
    """
    T = np.zeros((P, P))
    ntens = 1 + (P - 9) // 6  # stress + memory-variable tensors
    for col in range(P):
        e = np.zeros(P)
        e[col] = 1.0
        out = np.zeros(P)
        for blk in range(ntens):
            base = 0 if blk == 0 else 9 + 6 * (blk - 1)
            S = np.zeros((3, 3))
            for v, (i, j) in enumerate(VOIGT):
                S[i, j] = S[j, i] = e[base + v]
            Sg = R @ S @ R.T
            for v, (i, j) in enumerate(VOIGT):
                out[base + v] = Sg[i, j]
        out[6:9] = R @ e[6:9]
        T[:, col] = out
    return T


def godunov_state(Zp_m, Zs_m, Zp_p, Zs_p, P=9):
    """(G-, G+) in the face frame: q* = G- q- + G+ q+ (reading R8).

    Pairs (stress, velocity) on the normal axis x: (sxx, u) with Zp, (sxy, v) and (sxz, w)
    with Zs.  With Z- local and Z+ neighbour impedances:
        v*     = (Z- v- + Z+ v+ + s+ - s-) / (Z- + Z+)
        sigma* = (Z+ s- + Z- s+ + Z- Z+ (v+ - v-)) / (Z- + Z+)
    Components that the x-Jacobian does not read (syy, szz, syz, memory variables) are
    taken from the local side.
    """
    Gm = np.zeros((P, P))
    Gp = np.zeros((P, P))
    for sidx, vidx, Zm, Zpl in ((0, 6, Zp_m, Zp_p), (3, 7, Zs_m, Zs_p), (5, 8, Zs_m, Zs_p)):
        den = Zm + Zpl
        # v*
        Gm[vidx, vidx] = Zm / den
        Gp[vidx, vidx] = Zpl / den
        Gm[vidx, sidx] = -1.0 / den
        Gp[vidx, sidx] = 1.0 / den
        # sigma*
        Gm[sidx, sidx] = Zpl / den
        Gp[sidx, sidx] = Zm / den
        Gm[sidx, vidx] = -Zm * Zpl / den
        Gp[sidx, vidx] = Zm * Zpl / den
    for other in [1, 2, 4] + list(range(9, P)):
        Gm[other, other] = 1.0
    return Gm, Gp


def flux_solvers(n, mat_m, mat_p, P=9, omega=None):
    """(A+, A-) for a face with outward unit normal n (reading R8).

    mat = (rho, lam, mu).  F* = A+ q- + A- q+ approximates A_n(m-) q at the interface,
    with A_n = sum_d n_d A^d.  Signs and the face scaling are applied by the step.
    """
    rho_m, lam_m, mu_m = mat_m
    rho_p, lam_p, mu_p = mat_p
    R = face_frame(n)
    T = rotation(R, P)
    Tinv = rotation(R.T, P)
    Ahat = jacobians(rho_m, lam_m, mu_m, P, omega)[0]
    Zp_m = np.sqrt(rho_m * (lam_m + 2 * mu_m))
    Zs_m = np.sqrt(rho_m * mu_m)
    Zp_p = np.sqrt(rho_p * (lam_p + 2 * mu_p))
    Zs_p = np.sqrt(rho_p * mu_p)
    Gm, Gp = godunov_state(Zp_m, Zs_m, Zp_p, Zs_p, P)
    return T @ Ahat @ Gm @ Tinv, T @ Ahat @ Gp @ Tinv
