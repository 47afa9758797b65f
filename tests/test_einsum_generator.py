"""NEXT-4: the einsum front end of the generator (gen/einsum.py) -- EQSPP and strength
reduction -- against brute force and against what the paper states about its own kernels.

* EQSPP: zeroing a factor outside its EQSPP leaves the product unchanged, and
  every kept entry changes it for random values (brute force); the CK staircase
  C(N - d + 3, 3); the volume term's reduced GEMM saves 3/(N+3) of the flops,
  50 % at N = 3 and 37.5 % at N = 5 (reading R3).
* strength reduction: the dynamic program equals exhaustive enumeration of all
  evaluation trees on random sparse chains; the paper's neighbour-flux order
  R^((f(R I))A-) is optimal on the library's matrices; the factored chain beats applying the
  assembled B x B flux matrix by a factor growing linearly in N (O(N^6) -> O(N^5)).
* the generator consumes the front end: the emitted sources are unchanged when regenerated.
"""
import itertools
import os
import subprocess
import sys
from math import comb

import numpy as np
import pytest

from paper_1903_11521_b200.gen import einsum as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parse():
    out, idx, terms = E.parse("Q[kp] += Kh[ckl] I[lq] As[cpq]")
    assert (out, idx) == ("Q", "kp") and terms == [("Kh", "ckl"), ("I", "lq"), ("As", "cpq")]
    for bad in ("Q[kp] += Kh[ckl] I[lq", "Q += Kh[kl]", "Q[kp] = 3 * K[kp]"):
        with pytest.raises(ValueError):
            E.parse(bad)


def _rand_ops(rng, spec, density):
    """spec: [(name, idx)], sizes per index letter; random patterns and values."""
    sizes = {c: int(rng.integers(2, 5)) for c in "abcdefgh"}
    ops, vals = [], []
    for name, idx in spec:
        shape = tuple(sizes[c] for c in idx)
        pat = rng.random(shape) < density
        ops.append(E.Tensor(name, idx, pat))
        vals.append(np.where(pat, rng.standard_normal(shape), 0.0))
    return ops, vals


def _eval(ops, vals, out):
    args = []
    for t, v in zip(ops, vals):
        args += [v, [ord(c) - 97 for c in t.idx]]
    return np.einsum(*args, [ord(c) - 97 for c in out])


@pytest.mark.parametrize("seed", range(12))
def test_eqspp_brute_force(seed):
    rng = np.random.default_rng(seed)
    spec = [("A", "ab"), ("B", "bc"), ("C", "cd")] if seed % 2 else [("A", "abc"), ("B", "cd"), ("C", "bde")]
    out = "ad" if seed % 2 else "ae"
    ops, vals = _rand_ops(rng, spec, 0.4)
    red, res_pat = E.eqspp(ops, out)
    ref = _eval(ops, vals, out)
    # zeroing outside the EQSPP does not change the result
    vz = [np.where(r.pat, v, 0.0) for r, v in zip(red, vals)]
    assert np.allclose(_eval(ops, vz, out), ref, atol=1e-12)
    assert np.array_equal(res_pat, E.product_pattern(ops, out))
    # minimality: every kept entry changes the result when perturbed alone
    for i, r in enumerate(red):
        for pos in zip(*np.nonzero(r.pat)):
            v2 = [v.copy() for v in vals]
            v2[i][pos] += 1.0 + abs(v2[i][pos])
            assert not np.allclose(_eval(ops, v2, out), ref, atol=1e-12, rtol=0), (i, pos)


def _all_trees(items):
    if len(items) == 1:
        yield items[0]
        return
    first = items[0]
    rest = items[1:]
    for k in range(len(rest)):
        for left_rest in itertools.combinations(rest, k):
            left = (first,) + left_rest
            right = tuple(x for x in rest if x not in left_rest)
            if not right:
                continue
            for tl in _all_trees(left):
                for tr in _all_trees(right):
                    yield (tl, tr)


def _tree_cost(tree, ops, out):
    """Brute-force cost of an evaluation tree: nonzero multiply-adds of each binary
    contraction on the forward patterns (independent of the dynamic program)."""
    def leaves(t):
        return [t] if isinstance(t, int) else leaves(t[0]) + leaves(t[1])
    allidx = set(out)

    def go(t):
        if isinstance(t, int):
            return 0, ops[t]
        ca, A = go(t[0])
        cb, B = go(t[1])
        inside = set(leaves(t))
        outside = allidx | {c for j, o in enumerate(ops) if j not in inside for c in o.idx}
        keep = "".join(sorted({c for c in A.idx + B.idx if c in outside}))
        n = int(np.einsum(A.pat.astype(np.int64), [ord(c) - 97 for c in A.idx],
                          B.pat.astype(np.int64), [ord(c) - 97 for c in B.idx], []))
        pat = np.einsum(A.pat.astype(np.int64), [ord(c) - 97 for c in A.idx],
                        B.pat.astype(np.int64), [ord(c) - 97 for c in B.idx],
                        [ord(c) - 97 for c in keep]) > 0
        return ca + cb + 2 * n, E.Tensor("t", keep, pat)
    return go(tree)[0]


@pytest.mark.parametrize("seed", range(8))
def test_strength_reduction_equals_exhaustive_search(seed):
    rng = np.random.default_rng(100 + seed)
    spec = [("A", "ab"), ("B", "bc"), ("C", "cd"), ("D", "de")][: 3 + seed % 2]
    out = "a" + spec[-1][1][-1]
    ops, _ = _rand_ops(rng, spec, 0.5)
    red, _ = E.eqspp(ops, out)
    fl, tree = E.strength_reduce(ops, out)
    costs = [_tree_cost(t, red, out) for t in _all_trees(tuple(range(len(ops))))]
    assert fl == min(costs)
    assert _tree_cost(tree, red, out) == fl


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6])
def test_ck_staircase_and_volume_eqspp(N):
    """D^d has C(N-d+3,3) nonzero rows; reading R3: the volume term reads
    C(N+2,3) rows of I."""
    for d in range(N):
        assert E.ck_dims(N, d) == (comb(N - d + 3, 3), comb(N - d + 2, 3))
    assert E.vol_dim(N) == comb(N + 2, 3)
    pats = E.derivative_patterns(N)
    assert [int(p.any(axis=1).sum()) for p in pats] == [comb(N - d + 3, 3) for d in range(N + 1)]
    assert not pats[N][1:].any()  # D^N: the constant mode only


def test_volume_gemm_saving():
    """the EQSPP of I turns the (S, B, B) GEMM of the volume term into (S, B,
    Bv); the saving is 3/(N+3): 50 % for a fourth-order (N = 3), 37.5 % for a sixth-order
    (N = 5) scheme."""
    for N in range(1, 7):
        B = comb(N + 3, 3)
        saved = 1 - E.vol_dim(N) / B
        assert abs(saved - 3 / (N + 3)) < 1e-15
    assert 1 - E.vol_dim(3) / comb(6, 3) == 0.5
    assert 1 - E.vol_dim(5) / comb(8, 3) == 0.375


def _paper_order_cost(N, face, nface, h):
    """Cost of the paper's neighbour-flux order R^_ka ((f_ab (R_lb I_lq)) A-_pq)."""
    ops = E.operands("neighbour_flux", N, face=face, nface=nface, h=h)
    red, _ = E.eqspp(ops, "kp")
    # factor order in KERNELS: Rh, f, Rn, In, Am
    tree = (0, ((1, (2, 3)), 4))
    return _tree_cost(tree, red, "kp")


@pytest.mark.parametrize("case", [(3, 3, 0), (0, 2, 1), (2, 1, 2), (1, 0, 0)])
def test_paper_neighbour_flux_order_is_optimal(case):
    """R^((f(R I))A-) is an optimal order of the neighbour flux (single
    simulation); f and A- act on different indices, so applying them in either order after
    R I costs the same -- compare costs, not trees."""
    i, j, h = case
    ops = E.operands("neighbour_flux", 5, face=i, nface=j, h=h)
    fl, tree = E.strength_reduce(ops, "kp")
    assert fl == _paper_order_cost(5, i, j, h)


def test_strength_reduction_n6_to_n5():
    """the chain order reduces the neighbour flux from O(N^6) (the assembled
    B x B matrix R^ f R^T applied to I) to O(N^5): the ratio grows linearly in N."""
    ratios = []
    for N in (2, 3, 4, 5):
        ops = E.operands("neighbour_flux", N)
        fl, _ = E.strength_reduce(ops, "kp")
        K, R, f, B, Bt = E._mats(N)
        F = (R[3].astype(int) @ f[0].astype(int) @ R[3].T.astype(int)) > 0
        ratios.append((2 * int(F.sum()) * 9 + 2 * B * 81) / fl)
    steps = np.diff(ratios)
    assert (steps > 0.2).all() and (steps < 0.45).all(), ratios


def test_fused_simulations_merge_a_constant_pair():
    """with 8-32 fused simulations the optimal order contracts a pair of
    constant matrices before the simulation-dependent chain (the paper: R^ f).  On the
    library's matrices the merged pair is R^ f or f R depending on the face (DESIGN.md
    reading R28); either way the S-independent product appears and the order differs from
    the single-simulation one."""
    i, j, h = 0, 3, 0
    o1, _ = E.flux_chain_order(5, 1, face=i, nface=j, h=h)
    o8, f8 = E.flux_chain_order(5, 8, face=i, nface=j, h=h)
    assert "(Rh_ka f_ab)" in o8 or "(f_ab Rn_lb)" in o8, o8
    assert o1 != o8.replace("In_slq", "In_lq")


def test_generator_consumes_front_end():
    """gen/dmma.py, gen/kernels.py and gen/tiling.py take their product shapes from the
    front end; regenerating reproduces the committed sources byte for byte."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    for mod in ("paper_1903_11521_b200.gen.dmma", "paper_1903_11521_b200.gen.kernels"):
        subprocess.run([sys.executable, "-m", mod], cwd=ROOT, env=env, check=True, capture_output=True)
    r = subprocess.run(["git", "status", "--porcelain", "paper_1903_11521_b200/csrc/generated"],
                       cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("not a git checkout")
    assert r.stdout.strip() == "", r.stdout
