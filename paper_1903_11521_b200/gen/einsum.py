"""Einsum front end of the kernel generator (library side).

The kernels of the ADER-DG update are written here in the paper's index notation
 and analysed the way YATeTo does before it emits code:

* **equivalent sparsity patterns** (EQSPP): the smallest pattern of every
  tensor of a product such that zeroing the entries outside it does not change the result,
  found by propagating the nonzero patterns forward (which entries of the result can be
  nonzero) and backward (which entries of a factor meet a nonzero partner and a used entry of
  the result) to a fixed point -- this is what yields the staircase of the Cauchy-Kovalewski
  derivatives, C(N - delta + 3, 3) nonzero rows of D^delta, and the reduced
  GEMM of the volume term;
* **strength reduction** (P:1391-1400): the evaluation order of a multi-factor product by
  dynamic programming over subsets of its factors, minimising the nonzero flops of the
  binary contractions (2 per nonzero multiply-add, sparsity of every intermediate from its
  EQSPP).  It reproduces the paper's optimal chain for the neighbour flux,
  R^_ka ((f_ab (R_lb I_lq)) A-_pq), and for several fused simulations the order
  (R^_ka f_ab)((R_lb I_slq) A-_pq).

``plan(N)`` returns the products the GPU generator emits (gen/tiling.py, gen/dmma.py):
their operand patterns and shapes come from this analysis rather than from hand-written
closed forms.  The global matrices are the library's own (gen/tables.py); nothing here
touches the oracle.

    python -m paper_1903_11521_b200.gen.einsum [N]     # print the plan and the chain orders
"""
from __future__ import annotations

import itertools
import re
import sys
from functools import lru_cache

import numpy as np

from . import tables


class Tensor:
    """A named operand with one letter per index and a boolean nonzero pattern."""

    def __init__(self, name, idx, pattern):
        self.name, self.idx = name, idx
        self.pat = np.asarray(pattern, dtype=bool)
        assert self.pat.ndim == len(idx), (name, idx, self.pat.shape)

    def __repr__(self):
        return f"{self.name}[{self.idx}]{self.pat.shape}"


_TERM = re.compile(r"([A-Za-z_][A-Za-z0-9_]*)\[([a-z]*)\]")


def parse(expr):
    """'Q[kp] += Kh[ckl] I[lq] As[cpq]' -> (output name, output indices, [(name, indices)]).

    Einstein convention: an index that does not appear in the output is summed."""
    lhs, rhs = re.split(r"\+?=", expr, maxsplit=1)
    out = _TERM.fullmatch(lhs.strip())
    if out is None:
        raise ValueError(f"bad left-hand side: {lhs!r}")
    terms = _TERM.findall(rhs)
    if not terms or "".join(f"{n}[{i}]" for n, i in terms) != re.sub(r"\s+", "", rhs):
        raise ValueError(f"bad right-hand side: {rhs!r}")
    return out.group(1), out.group(2), terms


def _count(ops, out_idx=""):
    """Sum over all index assignments of the product of the 0/1 patterns (int64)."""
    ix = lambda s: [ord(c) - ord("a") for c in s]
    args = []
    for t in ops:
        args += [t.pat.astype(np.int64), ix(t.idx)]
    return np.einsum(*args, ix(out_idx), optimize=True)


def product_pattern(ops, out_idx):
    """Forward propagation: entries of the result that can be nonzero."""
    return _count(ops, out_idx) > 0


def eqspp(ops, out_idx, out_used=None):
    """Equivalent sparsity patterns of the factors of sum_(summed) prod(ops) -> out_idx.

    A factor entry is kept iff it is nonzero and, for some assignment of the other indices,
    every other factor is nonzero there and the result entry is used (out_used; default: the
    forward pattern).  Iterated to a fixed point (a pruned factor can prune another)."""
    ops = [Tensor(t.name, t.idx, t.pat.copy()) for t in ops]
    used = product_pattern(ops, out_idx) if out_used is None else np.asarray(out_used, bool)
    guard = Tensor("_out", out_idx, used)
    while True:
        changed = False
        for i, t in enumerate(ops):
            others = [o for j, o in enumerate(ops) if j != i] + [guard]
            reach = _count(others, t.idx) > 0 if others else np.ones_like(t.pat)
            new = t.pat & reach
            if not np.array_equal(new, t.pat):
                t.pat, changed = new, True
        if not changed:
            return ops, product_pattern(ops, out_idx) & used


def contraction_flops(a, b, keep):
    """Nonzero flops of the binary contraction a x b keeping the indices `keep`: one multiply
    and one add per nonzero product ('non-zero flops')."""
    return 2 * int(_count([a, b], ""))


def strength_reduce(ops, out_idx):
    """Optimal evaluation order of sum prod(ops) -> out_idx by dynamic programming over
    subsets of factors (the matrix-chain problem generalised to tensors).

    Returns (flops, tree) with tree = factor index or (left tree, right tree)."""
    ops, _ = eqspp(ops, out_idx)
    n = len(ops)
    best = {}  # frozenset -> (flops, tree, Tensor of the intermediate)
    for i, t in enumerate(ops):
        best[frozenset([i])] = (0, i, t)
    full = frozenset(range(n))
    for size in range(2, n + 1):
        for sub in itertools.combinations(range(n), size):
            sub = frozenset(sub)
            rest = full - sub
            # indices the intermediate of `sub` must keep: used outside it or in the output
            outside = set(out_idx) | {c for j in rest for c in ops[j].idx}
            cand = None
            for k in range(1, size // 2 + 1):
                for left in itertools.combinations(sorted(sub), k):
                    left = frozenset(left)
                    right = sub - left
                    if k * 2 == size and min(left) > min(right):
                        continue  # each split once
                    fl, tl, A = best[left]
                    fr, tr, Bt = best[right]
                    keep = "".join(sorted({c for c in A.idx + Bt.idx if c in outside}))
                    f = fl + fr + contraction_flops(A, Bt, keep)
                    if cand is None or f < cand[0]:
                        pat = product_pattern([A, Bt], keep)
                        cand = (f, (tl, tr), Tensor("(" + A.name + Bt.name + ")", keep, pat))
            best[sub] = cand
    f, tree, res = best[full]
    return f, tree


def tree_str(tree, ops):
    if isinstance(tree, int):
        t = ops[tree]
        return f"{t.name}_{t.idx}"
    return "(" + " ".join(tree_str(t, ops) for t in tree) + ")"


# ---------------------------------------------------------------------------------------
# the kernels of P:1312-1342 on the library's global matrices

@lru_cache(maxsize=None)
def _mats(N):
    t = tables.load(N)
    K = np.array(t["K"], dtype=float)      # K^c_kl, c = xi, eta, zeta
    R = np.array(t["R"], dtype=float)      # R^i_ka (B x Bt)
    f = np.array(t["f"], dtype=float)      # f^h_ab (Bt x Bt)
    return K != 0, R != 0, f != 0, t["B"], t["Bt"]


# star matrices A*^c (9 x 9): stresses read velocities, velocities read stresses
# (setup.cpp star_cols); the flux solvers A+- are dense 9 x 9
_STAR_COLS = ((6, 7, 8), (6, 7, 8), (6, 7, 8), (6, 7), (7, 8), (6, 8), (0, 3, 5), (3, 1, 4), (5, 4, 2))


def star_pattern():
    A = np.zeros((3, 9, 9), bool)
    for p, cols in enumerate(_STAR_COLS):
        A[:, p, list(cols)] = True
    return A


KERNELS = {
    # D^{d+1}_kp = sum_c Kt^c_kl D^d_lq A*^c_pq,  Kt^c = -K^cT
    "derivative": "D1[kp] = Kt[ckl] D0[lq] As[cpq]",
    # Q_kp += sum_c Kh^c_kl I_lq A*^c_pq,  Kh^c = K^c
    "volume": "Q[kp] += Kh[ckl] I[lq] As[cpq]",
    # local flux Q += R^_ka (R_la I_lq) A+_pq (face i; R^ = R up to M^-1, same pattern)
    "local_flux": "Q[kp] += Rh[ka] R[la] I[lq] Ap[pq]",
    # neighbour flux Q += R^_ka f_ab R'_lb I'_lq A-_pq (neighbour's face j, orientation h)
    "neighbour_flux": "Q[kp] += Rh[ka] f[ab] Rn[lb] In[lq] Am[pq]",
    # P:1306-1308 with the index s of fused simulations
    "neighbour_flux_fused": "Q[skp] += Rh[ka] f[ab] Rn[lb] In[slq] Am[pq]",
}


def operands(name, N, face=3, nface=3, h=0, S=8, dpat=None):
    """Tensors of kernel `name` at order N (face i, neighbour face j, orientation h)."""
    K, R, f, B, Bt = _mats(N)
    A = star_pattern()
    dense9 = np.ones((9, 9), bool)
    full = lambda *shape: np.ones(shape, bool)
    table = {
        "Kt": K.transpose(0, 2, 1), "Kh": K, "As": A,
        "D0": full(B, 9) if dpat is None else dpat, "I": full(B, 9), "In": full(B, 9),
        "Rh": R[face], "R": R[face], "Rn": R[nface], "f": f[h], "Ap": dense9, "Am": dense9,
    }
    if name.endswith("_fused"):
        table["In"] = full(S, B, 9)
    _, _, terms = parse(KERNELS[name])
    return [Tensor(n, i, table[n]) for n, i in terms]


def derivative_patterns(N):
    """Nonzero patterns of D^0..D^N of the Cauchy-Kovalewski recursion (P:1366-1369 and the
    paper's Fig. automatic_derivative_spp): D^0 = Q dense, D^{d+1} = forward pattern of the
    derivative kernel applied to D^d."""
    out_name, out_idx, _ = parse(KERNELS["derivative"])
    pats = [np.ones((_mats(N)[3], 9), bool)]
    for _ in range(N):
        ops = operands("derivative", N, dpat=pats[-1])
        pats.append(product_pattern(ops, out_idx))
    return pats


def rows_of(pat):
    """Rows of a [row][quantity] pattern with any nonzero (the EQSPP row set)."""
    return [int(r) for r in np.flatnonzero(pat.any(axis=1))]


@lru_cache(maxsize=None)
def shapes(N):
    """EQSPP-derived row sets of the products the GPU generator emits.

    ck[d] = (input rows of D^d, output rows of D^{d+1}) of CK step d; vol = input rows of
    the time integral the volume term reads (the nonzero columns of the EQSPP of Kh)."""
    pats = derivative_patterns(N)
    ck = []
    for d in range(N):
        ins, outs = rows_of(pats[d]), rows_of(pats[d + 1])
        # the product's EQSPP: only the rows of Kt that meet D^d's rows matter
        ops, res = eqspp(operands("derivative", N, dpat=pats[d]), "kp")
        assert rows_of(res) == outs
        ck.append((ins, outs))
    ops, _ = eqspp(operands("volume", N), "kp")
    vol = [int(l) for l in np.flatnonzero(ops[0].pat.any(axis=(0, 1)))]
    return {"ck": ck, "vol": vol}


def _leading(rows):
    # the kernels address the nonzero rows of D^d / I as the leading rows of their buffers
    # (degree-ordered basis, reading R6); the EQSPP must agree
    assert rows == list(range(len(rows))), rows
    return len(rows)


def ck_dims(N, d):
    """(rows in, rows out) of CK step d, from the EQSPP."""
    ins, outs = shapes(N)["ck"][d]
    return _leading(ins), _leading(outs)


def vol_dim(N):
    """Rows of the time integral the volume term reads (reading R3), from the EQSPP."""
    return _leading(shapes(N)["vol"])


@lru_cache(maxsize=None)
def plan(N):
    """shapes(N) plus orders = the strength-reduced evaluation order of every kernel."""
    sh = shapes(N)
    ck, vol = sh["ck"], sh["vol"]
    pats = derivative_patterns(N)
    orders = {}
    for name in ("derivative", "volume", "local_flux", "neighbour_flux"):
        ops = operands(name, N, dpat=pats[0] if name == "derivative" else None)
        fl, tree = strength_reduce(ops, parse(KERNELS[name])[1])
        orders[name] = (tree_str(tree, ops), fl)
    return {"ck": ck, "vol": vol, "orders": orders}


def flux_chain_order(N, S=1, face=3, nface=3, h=0):
    """Strength-reduced order (and nonzero flops) of the neighbour flux chain for S fused
    simulations (S = 1: the single-simulation kernel)."""
    name = "neighbour_flux" if S == 1 else "neighbour_flux_fused"
    ops = operands(name, N, face=face, nface=nface, h=h, S=S)
    fl, tree = strength_reduce(ops, parse(KERNELS[name])[1])
    return tree_str(tree, ops), fl


def main(argv):
    Ns = [int(a) for a in argv] or [5]
    for N in Ns:
        p = plan(N)
        print(f"N = {N}")
        for d, (i, o) in enumerate(p["ck"]):
            print(f"  CK step {d}: rows in {len(i)}, rows out {len(o)}")
        print(f"  volume reads {len(p['vol'])} rows of I")
        for k, (o, fl) in p["orders"].items():
            print(f"  {k}: {o}  ({fl} nonzero flops)")
        for S in (1, 8, 16, 32):
            o, fl = flux_chain_order(N, S)
            print(f"  neighbour flux, S = {S}: {o}  ({fl} nonzero flops)")


if __name__ == "__main__":
    main(sys.argv[1:])
