"""Local time stepping (LTS) of the ADER-DG scheme with two clusters, rate 2.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Row NEXT-2 of SURVEY §8(f).

The paper measures LTS against global time stepping on LOH.1 (Table loh1, P:1755-1769:
42.1 -> 17.8 min for DP; "LTS is less efficient due to smaller loop lengths, but pays off
in time-to-solution") but prints no LTS equations.  Reading R26,
the clustered ADER-DG LTS of the cited SeisSol scheme with two clusters and rate 2:
elements of cluster 0 ("fine") advance by dt, those of cluster 1 ("coarse") by 2 dt, and one
LTS cycle takes every element from t to t + 2 dt:

  coarse:  D^d from Q(t);  I_c = I[0, 2dt],  I_c1 = I[0, dt],  I_c2 = I[dt, 2dt]
  fine, substep k = 1, 2:  D^d from Q(t + (k-1) dt);  I_fk = I[0, dt]
           Q += volume(I_fk) + local flux(I_fk) + neighbour flux with, per face,
                I_fk of a fine neighbour or I_ck of a coarse neighbour
  coarse:  Q += volume(I_c) + local flux(I_c) + neighbour flux with, per face,
                I_c of a coarse neighbour or I_f1 + I_f2 of a fine neighbour

with the Taylor time integral over a sub-interval of the element's own expansion
  I[a, b] = sum_{d=0}^{N} (b^(d+1) - a^(d+1)) / (d+1)! D^d     (P:1326-1333 on [a, b]).
Every face flux of the step of P:1334-1342 thus integrates the neighbour's Taylor
expansion over exactly the interval the element advances, so the scheme reduces to global
time stepping when all elements share a cluster.
"""
from __future__ import annotations

from math import factorial

import numpy as np

from . import step


def interval_integral(Ds, a, b):
    """I[a, b] from the derivatives Ds = [D^0 .. D^N] (P:1326-1333 on [a, b])."""
    return sum((b ** (d + 1) - a ** (d + 1)) / factorial(d + 1) * D for d, D in enumerate(Ds))


def _derivatives(prob, Q):
    _, Ds = step.time_integral(prob, Q, 1.0)
    return Ds


def _update(prob, Q, sel, I_own, nb_integral):
    """Q^(n+1) for the elements `sel`: volume and local flux with I_own (E, B, P),
    neighbour flux of face i of element e with nb_integral(e, i) (B, P)."""
    out = Q.copy()
    for c in range(3):
        out[sel] += np.einsum("kl,elq->ekq", prob.Kh[c], I_own[sel]) @ np.transpose(prob.Astar[sel, c], (0, 2, 1))
    if prob.E_src is not None:
        out[sel] += I_own[sel] @ np.transpose(prob.E_src[sel], (0, 2, 1))
    for i in range(4):
        loc = np.einsum("kl,elq->ekq", prob.Fm[i], I_own[sel]) @ np.transpose(prob.Aplus[sel, i], (0, 2, 1))
        out[sel] -= prob.s[sel, i, None, None] * loc
    for e in sel:
        for i in range(4):
            Fp = prob.fp_mats[prob.fp_key[4 * e + i]]
            out[e] -= prob.s[e, i] * (Fp @ nb_integral(e, i) @ prob.Aminus[e, i].T)
    return out


def lts_cycle(prob: step.Problem, Q, dt, cluster):
    """One LTS cycle (t -> t + 2 dt); cluster[e] = 0 (dt) or 1 (2 dt); Q (E, B, P) internal."""
    cluster = np.asarray(cluster)
    fine = np.flatnonzero(cluster == 0)
    coarse = np.flatnonzero(cluster == 1)
    Dc = _derivatives(prob, Q)
    Ic = interval_integral(Dc, 0.0, 2 * dt)
    Ic1 = interval_integral(Dc, 0.0, dt)
    Ic2 = interval_integral(Dc, dt, 2 * dt)
    # fine substep 1
    Df = _derivatives(prob, Q)
    If1 = interval_integral(Df, 0.0, dt)
    Q1 = _update(prob, Q, fine, If1, lambda e, i: (If1 if cluster[prob.nb[e, i]] == 0 else Ic1)[prob.nb[e, i]])
    # fine substep 2 (derivatives of the fine elements at t + dt)
    Df2 = _derivatives(prob, Q1)
    If2 = interval_integral(Df2, 0.0, dt)
    Q2 = _update(prob, Q1, fine, If2, lambda e, i: (If2 if cluster[prob.nb[e, i]] == 0 else Ic2)[prob.nb[e, i]])
    # coarse step over 2 dt (its own state is still Q(t) in Q2)
    Ifs = If1 + If2
    Q3 = _update(prob, Q2, coarse, Ic, lambda e, i: (Ifs if cluster[prob.nb[e, i]] == 0 else Ic)[prob.nb[e, i]])
    return Q3


def lts(prob, Q, dt, cluster, ncycles=1):
    for _ in range(ncycles):
        Q = lts_cycle(prob, Q, dt, cluster)
    return Q
