"""Host-side checks of the kernel generators (no GPU): the annealed row groupings of
gen/tiling.py partition the rows, and the DMMA fragment tables emitted by gen/dmma.py
reproduce every global-matrix product exactly -- each nonzero lands in exactly one issued
8x4 tile and every skipped tile is zero (the zero-block exploitation must be exact)."""
import numpy as np
import pytest

from paper_1903_11521_b200.gen import dmma, tables, tiling


def _pad(g, n):
    return list(g) + [None] * (n - len(g))


def _rebuild(mats_shape, outs, ins, tab_frags, plan_tiles, which):
    """Dense matrix from the fragments of one matrix (index `which` in the product)."""
    M = np.zeros(mats_shape)
    hits = np.zeros(mats_shape, dtype=int)
    for (c, mt, tid, ks) in plan_tiles:
        if c != which:
            continue
        rows, cols = _pad(outs[mt], 8), _pad(ks, 4)
        fr = tab_frags[tid]
        for i in range(32):
            r, cc = rows[i // 4], cols[i % 4]
            if r is None or cc is None:
                assert fr[i] == 0.0
                continue
            M[r, cc] += fr[i]
            hits[r, cc] += 1
    return M, hits


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_tilings_partition_rows(N):
    til = tiling.tiling(N)
    for name, (mats, classes, *rest) in tiling.products(N).items():
        t = til[name]
        nout, nin = mats[0].shape
        assert sorted(r for g in t["out"] for r in g) == list(range(nout)), name
        assert all(len(g) <= 8 for g in t["out"])
        for part in t["in"]:
            assert sorted(r for g in part for r in g) == list(range(nin)), name
            assert all(len(g) <= 4 for g in part)
            for g in part:  # a k-set never mixes input-row classes
                assert sum(any(r in cl for r in g) for cl in classes) == 1, (name, g)


@pytest.mark.parametrize("N", [2, 5])
def test_dmma_fragments_reproduce_the_matrices(N):
    t = tables.load(N)
    K = [np.array(k) for k in t["K"]]
    til = tiling.tiling(N)
    from math import comb
    Bv = comb(N + 2, 3)
    cases = {"vol": ([K[c][:, :Bv] for c in range(3)], til["vol"])}
    for d in range(N):
        bi, bo = comb(N - d + 3, 3), comb(N - d + 2, 3)
        cases[f"ck{d}"] = ([-K[c].T[:bo, :bi] for c in range(3)], til[f"ck{d}"])
    for name, (mats, tl) in cases.items():
        tab = dmma.Table()
        funcs = [(lambda r, col, M=M: M[r, col]) for M in mats]
        plan = dmma.plan_xprod(tab, funcs, tl)
        tiles = [(c, mt, tid, ks) for ks, tl_ in zip(tl["in"][0], plan) for (c, mt, tid) in tl_]
        for which, M in enumerate(mats):
            R, hits = _rebuild(M.shape, tl["out"], tl["in"][0], tab.frags, tiles, which)
            assert np.array_equal(R, M), name
            assert hits.max() <= 1, name  # no entry covered twice
            assert np.all(hits[M != 0] == 1), name  # every nonzero issued
