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
    K = [np.array(k) for k in tables.kdir(t)]  # the kernels' derivative directions
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


def _setup_h_constants():
    """kDirT / kDirTinv as compiled into the library (csrc/setup.h)."""
    import os
    import re
    src = open(os.path.join(os.path.dirname(tables.__file__), "..", "csrc", "setup.h")).read()
    out = {}
    for name in ("kDirT", "kDirTinv"):
        body = re.search(name + r"\[3\]\[3\] = \{(.*?)\};", src, re.S).group(1)
        out[name] = np.array([float(v) for v in re.findall(r"-?\d+(?:\.\d+)?", body)]).reshape(3, 3)
    return out


def test_derivative_directions_are_an_exact_reformulation():
    """The kernels' K'^c = sum_d T_cd K^d with star matrices A*'^c = sum_d (T^-1)_dc A*^d give
    sum_c K'^c X A*'^c = sum_c K^c X A*^c for any X and star matrices: the library's
    constants (setup.h) are T and its inverse, and T equals gen/tables.py KDIR_T."""
    c = _setup_h_constants()
    T = np.array(tables.KDIR_T, dtype=float)
    assert np.array_equal(c["kDirT"], T)
    assert np.array_equal(c["kDirTinv"] @ T, np.eye(3)) and np.array_equal(T @ c["kDirTinv"], np.eye(3))
    rng = np.random.default_rng(7)
    for N in (2, 5):
        t = tables.load(N)
        K = np.array(t["K"])
        Kd = np.array(tables.kdir(t))
        X = rng.normal(size=(K.shape[1], 9))
        A = rng.normal(size=(3, 9, 9))
        Ad = np.einsum("dc,dpq->cpq", c["kDirTinv"], A)
        ref = sum(K[k] @ X @ A[k].T for k in range(3))
        got = sum(Kd[k] @ X @ Ad[k].T for k in range(3))
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        # the CK direction (Ktilde = -K^T) obeys the same identity
        ref = sum(-K[k].T @ X @ A[k].T for k in range(3))
        got = sum(-Kd[k].T @ X @ Ad[k].T for k in range(3))
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("N,nnz_ref,nnz_dir", [(2, 46, 29), (3, 202, 119), (4, 647, 364), (5, 1708, 924), (6, 3920, 2058)])
def test_derivative_directions_cut_the_nonzeros(N, nnz_ref, nnz_dir):
    """Nonzeros of the three derivative matrices in the reference directions and in KDIR_T's
    (exact zeros: the cancellations of the Dubiner structure are exact)."""
    t = tables.load(N)
    assert sum(int(np.count_nonzero(np.array(k))) for k in t["K"]) == nnz_ref
    Kd = tables.kdir(t)
    assert sum(int(np.count_nonzero(np.array(k))) for k in Kd) == nnz_dir
    # the staircase of the CK recursion survives: K'^c maps degree <= n to degree <= n - 1
    from math import comb
    Bv = comb(N + 2, 3)
    assert all(not np.any(np.array(k)[:, Bv:]) for k in Kd)


def test_c_annealer_agrees_with_the_tile_count_definition(tmp_path):
    """tools/anneal.c keeps the tile count incrementally; its reported cost must equal
    gen/tiling's definition (count of nonzero 8x4 blocks) on the groupings it returns, and
    reach the cached tile counts of a small order."""
    import importlib.util
    import os
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("reanneal", os.path.join(root, "tools", "reanneal.py"))
    re_ = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(re_)
    exe = str(tmp_path / "anneal")
    subprocess.run(["gcc", "-O2", "-o", exe, os.path.join(root, "tools", "anneal.c"), "-lm"], check=True)
    cached = tiling.tiling(3)
    for name, pr in tiling.products(3).items():
        if name not in ("ck0", "vol", "lift"):
            continue
        res, costs = re_.solve(name, pr, 200000, 4, exe, 2)  # solve() asserts cost == definition
        rows = sorted(r for g in res["out"] for r in g)
        assert rows == list(range(pr[0][0].shape[0]))
        assert res["tiles"] <= cached[name]["tiles"] + 1
