"""One ADER-DG step of the elastic / viscoelastic scheme, plain dense evaluation.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Scheme (with readings R1-R4, R8, R14 of DESIGN.md §3), per element e,
all elements using the same snapshot Q^n:

  D^0 = Q^n_e
  D^(d+1)_kp = sum_c sum_l sum_q Kt^c_kl D^d_lq A*^c_pq   (+ sum_q D^d_kq E_pq)
  I_e = sum_{d=0}^{N} dt^(d+1)/(d+1)! D^d
  Q^(n+1)_kp = Q^n_kp + sum_c sum_l sum_q Kh^c_kl I_lq A*^c_pq   (+ sum_q I_kq E_pq)
              - sum_i s_i sum_l sum_q Fm^i_kl I_lq (A+_i)_pq
              - sum_i s_i sum_l sum_q Fp^(e,i)_kl I^(nb)_lq (A-_i)_pq

with s_i = 2 |S_i| / det J (dS = 2|S_i| dchi dtau, dV = det J dxi), Fm^i and Fp^(e,i) the
*dense* B x B face matrices (no factorisation R f R^T, no sparsity), Fp built from the
vertex-id correspondence of the shared face (not from the (j, h) tables).  The paper folds
-s_i into its A+, A- (reading R4).  All arithmetic is fp64.

Layout: the public (canonical) DOF layout is [element][quantity][basis] (P = quantities,
B = basis functions); internally the oracle works on Q_kp = [element][basis][quantity].

``literal_update`` (tiny inputs only) re-evaluates every term as ONE multi-operand
Einstein sum over the full index space, exactly as written in P:1312-1342 including the
factored chain R f R I A- (P:1342), and is used to pin the index conventions.
"""
from __future__ import annotations

from dataclasses import dataclass
from math import factorial

import numpy as np

from . import matrices, mesh, physics


@dataclass
class Problem:
    """Everything the step needs, built from raw inputs by ``setup``."""
    N: int
    P: int
    Kt: np.ndarray        # (3, B, B)
    Kh: np.ndarray        # (3, B, B)
    Astar: np.ndarray     # (E, 3, P, P)
    E_src: np.ndarray     # (E, P, P) or None
    s: np.ndarray         # (E, 4) face scaling 2|S_i|/det J
    Aplus: np.ndarray     # (E, 4, P, P)
    Aminus: np.ndarray    # (E, 4, P, P)
    nb: np.ndarray        # (E, 4)
    fp_key: list          # per (e, i): key into fp_mats
    fp_mats: dict         # key -> (B, B) neighbour face matrix
    Fm: np.ndarray        # (4, B, B)


def setup(N, elem_xyz, elem_vid, mat, P=9, omega=None, Y=None, elements=None):
    """Build a Problem.  mat: (E,3) rho, vp, vs.  elements: optional subset (then the
    Problem covers only those elements, but neighbours index the full mesh)."""
    elem_xyz = np.asarray(elem_xyz, dtype=np.float64)
    elem_vid = np.asarray(elem_vid)
    Eall = elem_xyz.shape[0]
    sel = np.arange(Eall) if elements is None else np.asarray(elements)
    nb_all = mesh.match_faces(elem_vid) if elements is None else _match_faces_subset(elem_vid, sel)
    J, Jinv, detJ, area, normal = mesh.geometry(elem_xyz[sel])
    rho, vp, vs = mat[:, 0], mat[:, 1], mat[:, 2]
    lam, mu = physics.lame(rho, vp, vs)
    E = len(sel)
    Astar = np.zeros((E, 3, P, P))
    Esrc = np.zeros((E, P, P)) if P == 27 else None
    Aplus = np.zeros((E, 4, P, P))
    Aminus = np.zeros((E, 4, P, P))
    keys = []
    for n, e in enumerate(sel):
        A = physics.jacobians(rho[e], lam[e], mu[e], P, omega)
        Astar[n] = physics.star_matrices(Jinv[n], A)
        if P == 27:
            Esrc[n] = physics.source_matrix(omega, Y[e, :, 0], Y[e, :, 1])
        for i in range(4):
            o = nb_all[n, i]
            Ap, Am = physics.flux_solvers(normal[n, i], (rho[e], lam[e], mu[e]), (rho[o], lam[o], mu[o]), P, omega)
            Aplus[n, i] = Ap
            Aminus[n, i] = Am
            keys.append((matrices.FACES[i], mesh.neighbour_vertex_map(elem_vid, e, i, o)))
    fp_mats = {k: matrices.face_pair_matrix(N, k[0], k[1]) for k in set(keys)}
    s = 2.0 * area / detJ[:, None]
    Fm = np.array([matrices.face_mass_matrix(N, i) for i in range(4)])
    return Problem(N, P, matrices.derivative_matrices(N), matrices.volume_matrices(N), Astar, Esrc, s,
                   Aplus, Aminus, nb_all, keys, fp_mats, Fm)


def _match_faces_subset(elem_vid, sel):
    """Neighbours of the selected elements in the full mesh (vectorised key matching)."""
    vid = np.asarray(elem_vid, dtype=np.int64)
    E = vid.shape[0]
    m = int(vid.max()) + 1
    keys = np.zeros((E, 4), dtype=np.int64)
    for i, tri in enumerate(matrices.FACES):
        t = np.sort(vid[:, list(tri)], axis=1)
        keys[:, i] = (t[:, 0] * m + t[:, 1]) * m + t[:, 2]
    flat = keys.ravel()
    order = np.argsort(flat, kind="stable")
    sk = flat[order]
    if len(sk) % 2 or np.any(sk[0::2] != sk[1::2]) or np.any(sk[1:-1:2] == sk[2::2]):
        raise ValueError("face not matched exactly twice")
    partner = np.empty_like(order)
    partner[order[0::2]] = order[1::2]
    partner[order[1::2]] = order[0::2]
    nb = (partner // 4).reshape(E, 4)
    return nb[np.asarray(sel)]


def time_integral(prob: Problem, Q, dt):
    """(I, [D^0..D^N]) for Q (E, B, P) internal layout."""
    D = Q.copy()
    Ds = [D]
    I = dt * D
    for d in range(prob.N):
        Dn = np.zeros_like(D)
        for c in range(3):
            Dn += np.einsum("kl,elq->ekq", prob.Kt[c], D) @ np.transpose(prob.Astar[:, c], (0, 2, 1))
        if prob.E_src is not None:
            Dn += D @ np.transpose(prob.E_src, (0, 2, 1))
        D = Dn
        Ds.append(D)
        I = I + dt ** (d + 2) / factorial(d + 2) * D
    return I, Ds


def update(prob: Problem, Q, I, I_full=None):
    """Q^(n+1) = Q^n + volume + local flux + neighbour flux.

    Q, I: (E, B, P) for the problem's elements; I_full: time integrals of the full mesh
    (indexed by prob.nb); defaults to I (problem covers the full mesh)."""
    if I_full is None:
        I_full = I
    out = Q.copy()
    for c in range(3):
        out += np.einsum("kl,elq->ekq", prob.Kh[c], I) @ np.transpose(prob.Astar[:, c], (0, 2, 1))
    if prob.E_src is not None:
        out += I @ np.transpose(prob.E_src, (0, 2, 1))
    for i in range(4):
        loc = np.einsum("kl,elq->ekq", prob.Fm[i], I) @ np.transpose(prob.Aplus[:, i], (0, 2, 1))
        out -= prob.s[:, i, None, None] * loc
    E = Q.shape[0]
    for i in range(4):
        Inb = I_full[prob.nb[:, i]]
        nbt = np.zeros_like(Q)
        groups = {}
        for e in range(E):
            groups.setdefault(prob.fp_key[4 * e + i], []).append(e)
        for k, idx in groups.items():
            idx = np.array(idx)
            nbt[idx] = np.einsum("kl,elq->ekq", prob.fp_mats[k], Inb[idx])
        out -= prob.s[:, i, None, None] * (nbt @ np.transpose(prob.Aminus[:, i], (0, 2, 1)))
    return out


def step(prob: Problem, Q, dt, nsteps=1):
    """nsteps global time steps; Q (E, B, P) internal layout, full mesh."""
    for _ in range(nsteps):
        I, _ = time_integral(prob, Q, dt)
        Q = update(prob, Q, I)
    return Q


def to_internal(Qc):
    """canonical [e][p][k] -> internal [e][k][p]."""
    return np.ascontiguousarray(np.transpose(Qc, (0, 2, 1)))


def to_canonical(Q):
    return np.ascontiguousarray(np.transpose(Q, (0, 2, 1)))


def literal_update(prob: Problem, Q, dt, nbtab):
    """One step evaluated term by term as single Einstein sums (tiny inputs only).

    Uses the paper's factored neighbour chain  R^i_km f^h_mn R^j_ln I^nb_lq (A-)_pq
     with the oracle's brute-force (nb, j, h) tables ``nbtab`` and the local chain
    R^i_km R^i_lm I_lq (A+)_pq.  Returns Q^(n+1) (E, B, P).
    """
    N = prob.N
    nb, jj, hh = nbtab
    D = [Q]
    for d in range(N):
        t = np.einsum("ckl,elq,ecpq->ekp", prob.Kt, D[-1], prob.Astar)
        if prob.E_src is not None:
            t = t + np.einsum("ekq,epq->ekp", D[-1], prob.E_src)
        D.append(t)
    I = sum(dt ** (d + 1) / factorial(d + 1) * D[d] for d in range(N + 1))
    R = np.array([matrices.lift_matrix(N, i) for i in range(4)])
    f = np.array([matrices.rotation_matrix(N, h) for h in range(3)])
    out = Q + np.einsum("ckl,elq,ecpq->ekp", prob.Kh, I, prob.Astar)
    if prob.E_src is not None:
        out = out + np.einsum("ekq,epq->ekp", I, prob.E_src)
    out = out - np.einsum("ei,ikm,ilm,elq,eipq->ekp", prob.s, R, R, I, prob.Aplus)
    Rj = R[jj]            # (E, 4, B, Bt)
    fh = f[hh]            # (E, 4, Bt, Bt)
    Inb = I[nb]           # (E, 4, B, P)
    out = out - np.einsum("ei,ikm,eimn,eiln,eilq,eipq->ekp", prob.s, R, fh, Rj, Inb, prob.Aminus)
    return out


# ---- multiple fused simulations: the scheme with an extra index s
# on the degrees of freedom Q_skp, the derivatives D_skp and the time integral I_skp; every
# matrix (global, star, flux) is shared by the S simulations.

def time_integral_fused(prob: Problem, Q, dt):
    """(I, [D^0..D^N]) for Q (S, E, B, P):  D^(d+1)_sekp = sum_c Kt^c_kl D^d_selq A*^c_epq."""
    D = Q.copy()
    Ds = [D]
    I = dt * D
    for d in range(prob.N):
        Dn = np.zeros_like(D)
        for c in range(3):
            Dn += np.einsum("kl,selq,epq->sekp", prob.Kt[c], D, prob.Astar[:, c])
        if prob.E_src is not None:
            Dn += np.einsum("sekq,epq->sekp", D, prob.E_src)
        D = Dn
        Ds.append(D)
        I = I + dt ** (d + 2) / factorial(d + 2) * D
    return I, Ds


def update_fused(prob: Problem, Q, I):
    """Q^(n+1)_sekp (P:1334-1342 with the index s); Q, I: (S, E, B, P), full mesh."""
    out = Q.copy()
    for c in range(3):
        out += np.einsum("kl,selq,epq->sekp", prob.Kh[c], I, prob.Astar[:, c])
    if prob.E_src is not None:
        out += np.einsum("sekq,epq->sekp", I, prob.E_src)
    for i in range(4):
        out -= np.einsum("e,kl,selq,epq->sekp", prob.s[:, i], prob.Fm[i], I, prob.Aplus[:, i])
    E = Q.shape[1]
    for i in range(4):
        Inb = I[:, prob.nb[:, i]]
        for e in range(E):
            Fp = prob.fp_mats[prob.fp_key[4 * e + i]]
            out[:, e] -= prob.s[e, i] * np.einsum("kl,slq,pq->skp", Fp, Inb[:, e], prob.Aminus[e, i])
    return out


def step_fused(prob: Problem, Q, dt, nsteps=1):
    """nsteps global time steps of S fused simulations; Q (S, E, B, P) internal layout."""
    for _ in range(nsteps):
        I, _ = time_integral_fused(prob, Q, dt)
        Q = update_fused(prob, Q, I)
    return Q
