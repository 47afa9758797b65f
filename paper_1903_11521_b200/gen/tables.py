"""Global matrices of the ADER-DG scheme for the CUDA path (library side).

Computes, in 40-digit arithmetic, the reference-element matrices the kernels hard-code
(the analogue of YATeTo's compile-time matrices "stored within the generated code",
P:1239-1241):

  K^c_kl  = int_T (d phi_k/d xi_c) phi_l   -> Ktilde^c = -K^cT, Khat^c = K^c
  R^i_km  = int_tri phi_k(x^(i)(chi,tau)) psi_m lift / trace projection
  f^h_mn  = int_tri psi_m psi_n(chit^h)      neighbour orientation

This is an independent construction from the oracle's: numerical Gauss quadrature in
collapsed coordinates with Jacobi three-term recurrences, gradients by the chain rule in
collapsed coordinates, all in mpmath at 40 digits, rounded once to fp64.  Conventions
(basis order, face triples, orientation maps) follow DESIGN.md §3 (readings R6, R7).

Run as a script to regenerate ``csrc/generated/ydg_matrices.h``.
"""
from __future__ import annotations

import os
from functools import lru_cache

import mpmath as mp

mp.mp.dps = 40

FACES = ((0, 2, 1), (0, 1, 3), (0, 3, 2), (1, 2, 3))
VERTS = ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1))


def jacobi(n, a, b, x):
    """P_n^(a,b)(x) by the three-term recurrence."""
    if n == 0:
        return mp.mpf(1)
    p0 = mp.mpf(1)
    p1 = (a + 1) + (a + b + 2) * (x - 1) / 2
    for k in range(2, n + 1):
        c1 = 2 * k * (k + a + b) * (2 * k + a + b - 2)
        c2 = (2 * k + a + b - 1) * (a * a - b * b)
        c3 = (2 * k + a + b - 2) * (2 * k + a + b - 1) * (2 * k + a + b)
        c4 = 2 * (k + a - 1) * (k + b - 1) * (2 * k + a + b)
        p0, p1 = p1, ((c2 + c3 * x) * p1 - c4 * p0) / c1
    return p1


def djacobi(n, a, b, x):
    return mp.mpf(0) if n == 0 else mp.mpf(n + a + b + 1) / 2 * jacobi(n - 1, a + 1, b + 1, x)


@lru_cache(maxsize=None)
def gauss_legendre(n):
    """Nodes/weights on [-1, 1] by Newton iteration on P_n."""
    xs, ws = [], []
    for i in range(1, n + 1):
        x = mp.cos(mp.pi * (i - mp.mpf(1) / 4) / (n + mp.mpf(1) / 2))
        for _ in range(100):
            p = jacobi(n, 0, 0, x)
            dp = djacobi(n, 0, 0, x)
            dx = p / dp
            x -= dx
            if abs(dx) < mp.mpf(10) ** (-mp.mp.dps + 3):
                break
        dp = djacobi(n, 0, 0, x)
        xs.append(x)
        ws.append(2 / ((1 - x * x) * dp * dp))
    return xs, ws


def tet_index(N):
    return [(d - q - r, q, r) for d in range(N + 1) for r in range(d + 1) for q in range(d - r + 1)]


def tri_index(N):
    return [(d - q, q) for d in range(N + 1) for q in range(d + 1)]


def phi_and_grad(p, q, r, xi, eta, zeta):
    """Unnormalised Dubiner function and its gradient at an interior point."""
    w1 = 1 - eta - zeta
    w2 = 1 - zeta
    a = 2 * xi / w1 - 1
    b = 2 * eta / w2 - 1
    c = 2 * zeta - 1
    al_b, al_c = 2 * p + 1, 2 * p + 2 * q + 2
    f = jacobi(p, 0, 0, a)
    df = djacobi(p, 0, 0, a)
    gb = ((1 - b) / 2) ** p
    g = gb * jacobi(q, al_b, 0, b)
    dg = gb * djacobi(q, al_b, 0, b) - (p * ((1 - b) / 2) ** (p - 1) / 2 * jacobi(q, al_b, 0, b) if p > 0 else 0)
    hc = ((1 - c) / 2) ** (p + q)
    h = hc * jacobi(r, al_c, 0, c)
    dh = hc * djacobi(r, al_c, 0, c) - ((p + q) * ((1 - c) / 2) ** (p + q - 1) / 2 * jacobi(r, al_c, 0, c) if p + q > 0 else 0)
    da = (2 / w1, 2 * xi / w1 ** 2, 2 * xi / w1 ** 2)
    db = (0, 2 / w2, 2 * eta / w2 ** 2)
    dc = (0, 0, 2)
    val = f * g * h
    grad = [df * g * h * da[k] + f * dg * h * db[k] + f * g * dh * dc[k] for k in range(3)]
    return val, grad


def psi(p, q, chi, tau):
    x = 2 * chi / (1 - tau) - 1
    return jacobi(p, 0, 0, x) * (1 - tau) ** p * jacobi(q, 2 * p + 1, 0, 2 * tau - 1)


@lru_cache(maxsize=None)
def tet_rule(n):
    xs, ws = gauss_legendre(n)
    pts = []
    for a, wa in zip(xs, ws):
        for b, wb in zip(xs, ws):
            for c, wc in zip(xs, ws):
                xi = (1 + a) * (1 - b) * (1 - c) / 8
                eta = (1 + b) * (1 - c) / 4
                zeta = (1 + c) / 2
                pts.append((xi, eta, zeta, wa * wb * wc * (1 - b) * (1 - c) ** 2 / 64))
    return pts


@lru_cache(maxsize=None)
def tri_rule(n):
    xs, ws = gauss_legendre(n)
    pts = []
    for a, wa in zip(xs, ws):
        for b, wb in zip(xs, ws):
            pts.append(((1 + a) * (1 - b) / 4, (1 + b) / 2, wa * wb * (1 - b) / 8))
    return pts


@lru_cache(maxsize=None)
def tables(N):
    """Dict of dense fp64 matrices (lists of lists): K (3,B,B), R (4,B,Bt), f (3,Bt,Bt)."""
    idx = tet_index(N)
    tidx = tri_index(N)
    B, Bt = len(idx), len(tidx)
    rule = tet_rule(N + 3)
    # basis values and gradients at the volume points
    vals = [[None] * len(rule) for _ in range(B)]
    grads = [[None] * len(rule) for _ in range(B)]
    for k, (p, q, r) in enumerate(idx):
        for s, (xi, eta, zeta, w) in enumerate(rule):
            v, g = phi_and_grad(p, q, r, xi, eta, zeta)
            vals[k][s], grads[k][s] = v, g
    norm = [1 / mp.sqrt(mp.fsum(vals[k][s] ** 2 * rule[s][3] for s in range(len(rule)))) for k in range(B)]
    K = [[[mp.fsum(grads[k][s][c] * vals[l][s] * rule[s][3] for s in range(len(rule))) * norm[k] * norm[l]
           for l in range(B)] for k in range(B)] for c in range(3)]
    trule = tri_rule(N + 2)
    tnorm = [1 / mp.sqrt(mp.fsum(psi(p, q, x, t) ** 2 * w for x, t, w in trule)) for p, q in tidx]
    psiv = [[psi(p, q, x, t) * tnorm[m] for x, t, w in trule] for m, (p, q) in enumerate(tidx)]
    R = []
    for (a, b, c) in FACES:
        Pa, Pb, Pc = VERTS[a], VERTS[b], VERTS[c]
        phis = []
        for x, t, w in trule:
            pt = [Pa[d] + x * (Pb[d] - Pa[d]) + t * (Pc[d] - Pa[d]) for d in range(3)]
            phis.append([phi_and_grad(*idx[k], *_interior(pt))[0] * norm[k] for k in range(B)])
        R.append([[mp.fsum(phis[s][k] * psiv[m][s] * trule[s][2] for s in range(len(trule)))
                   for m in range(Bt)] for k in range(B)])
    rots = (lambda x, t: (t, x), lambda x, t: (1 - x - t, t), lambda x, t: (x, 1 - x - t))
    f = []
    for rot in rots:
        rv = [[psi(p, q, *rot(x, t)) * tnorm[n] for x, t, w in trule] for n, (p, q) in enumerate(tidx)]
        f.append([[mp.fsum(psiv[m][s] * rv[n][s] * trule[s][2] for s in range(len(trule)))
                   for n in range(Bt)] for m in range(Bt)])
    clean = lambda v: 0.0 if abs(v) < mp.mpf(10) ** -25 else float(v)
    return {
        "K": [[[clean(v) for v in row] for row in Kc] for Kc in K],
        "R": [[[clean(v) for v in row] for row in Ri] for Ri in R],
        "f": [[[clean(v) for v in row] for row in fh] for fh in f],
        "B": B, "Bt": Bt,
    }


def _interior(pt):
    # face points of x = 0 style faces are interior to the face but may sit on the
    # collapse singularity only at vertices; Gauss points never do.
    return tuple(pt)


def _fmt(v):
    return repr(float(v)) if v != 0 else "0.0"


ORDERS = (1, 2, 3, 4, 5, 6)
JSON = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "csrc", "generated", "ydg_matrices.json")


def load(N):
    """Matrices of order N from the generated JSON (fast path for gen/kernels.py)."""
    import json
    if os.path.exists(JSON):
        with open(JSON) as fh:
            data = json.load(fh)
        if str(N) in data:
            return data[str(N)]
    return tables(N)


# Derivative directions of the kernels' CK and volume products: K'^c = sum_d KDIR_T[c][d] K^d,
# with the star matrices combined by the inverse (csrc/setup.h kDirT / kDirTinv, applied in
# setup.cpp), so that sum_c K'^c X A*'^c = sum_c K^c X A*^c.  The reference directions
# (1,0,0), (0,1,-1), (1,-2,0) minimise the nonzeros of the three matrices at every order
# N = 2..6 among integer directions with entries in [-3, 3] (N = 5: 924 instead of 1,708;
# tests/test_generator.py pins the identity and the counts).
KDIR_T = ((1, 0, 0), (0, 1, -1), (1, -2, 0))


def kdir(t):
    """K'^c[k][l] = sum_d KDIR_T[c][d] K^d[k][l]; sums that cancel exactly become exact zeros."""
    K = t["K"]
    B = len(K[0])
    out = []
    for c in range(3):
        M = []
        for k in range(B):
            row = []
            for l in range(B):
                v = sum(KDIR_T[c][d] * K[d][k][l] for d in range(3))
                m = max(abs(K[d][k][l]) for d in range(3))
                row.append(0.0 if abs(v) <= 1e-12 * m else v)
            M.append(row)
        out.append(M)
    return out


def emit_header(path, orders=ORDERS):
    lines = ["// GENERATED by paper_1903_11521_b200/gen/tables.py -- do not edit.",
             "// Reference-element matrices of the ADER-DG scheme (arXiv:1903.11521 Sec. 5.1),",
             "// dense row-major fp64: K[c][k][l] = int (d phi_k / d xi_c) phi_l, R[i][k][m], f[h][m][n].",
             "#pragma once", "namespace ydg { namespace tables {"]
    for N in orders:
        t = tables(N)
        B, Bt = t["B"], t["Bt"]
        lines.append(f"struct N{N} {{ static constexpr int B = {B}, Bt = {Bt};")
        for name, arr in (("K", t["K"]), ("R", t["R"]), ("f", t["f"])):
            flat = [_fmt(v) for m in arr for row in m for v in row]
            dims = f"[{len(arr)}][{len(arr[0])}][{len(arr[0][0])}]"
            lines.append(f"  static constexpr double {name}{dims} = {{")
            for s in range(0, len(flat), 6):
                lines.append("    " + ", ".join(flat[s:s + 6]) + ",")
            lines.append("  };")
        lines.append("};")
    lines.append("}}  // namespace ydg::tables")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    import json
    with open(JSON, "w") as fh:
        json.dump({str(N): tables(N) for N in orders}, fh)


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    out = os.path.join(here, "..", "csrc", "generated", "ydg_matrices.h")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    emit_header(out)
    print("wrote", out)
