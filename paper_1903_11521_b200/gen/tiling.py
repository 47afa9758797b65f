"""Row groupings of the global-matrix products for the DMMA m8n8k4 kernels.

A product Y (+)= M X with a sparse global matrix M (n_out x n_in; several matrices sharing
the output, e.g. the three K^c of one CK step) runs as 8x4 A-operand tiles.  The kernels
may gather ANY 8 output rows into an m-tile (the C fragments are scattered on write-back)
and ANY 4 input rows into a k-set (the B fragments / the star-matrix chunk X are built
from arbitrary rows), so the tile count is

    sum_c  #{ (m-tile, k-set) : M_c[m-tile rows, k-set rows] != 0 }

over a partition of the output rows into groups of 8 and of the input rows into groups of
4.  This is the zero-block exploitation of the paper's equivalent sparsity patterns
 with the block boundaries chosen freely instead of at fixed positions; the
partitions are found by simulated annealing (pairwise swaps) and cached in
``tilings/N<n>.json`` so that regeneration is deterministic and fast.

    python -m paper_1903_11521_b200.gen.tiling [--search N...]
"""
from __future__ import annotations

import json
import math
import os
import random
import sys

import numpy as np

from . import einsum, tables

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE_DIR = os.path.join(HERE, "tilings")


def products(N):
    """name -> (boolean patterns (n_out x n_in), input-row classes[, input partition of each]).

    Input-row classes: lists of input rows that may share a k-set (the trace products read
    rows < IROWS of the time integral from shared memory and the others, dt * Q, from global
    memory, so a k-set never mixes the two)."""
    t = tables.load(N)
    K = [np.array(k, dtype=float) != 0 for k in tables.kdir(t)]  # the kernels' directions (KDIR_T)
    R = [np.array(r, dtype=float) != 0 for r in t["R"]]
    B, Bt = t["B"], t["Bt"]
    Bv = einsum.vol_dim(N)
    irows = Bv  # rows of the time integral held in shared memory
    out = {}
    for d in range(N):
        bi, bo = einsum.ck_dims(N, d)
        out[f"ck{d}"] = ([K[c].T[:bo, :bi] for c in range(3)], [list(range(bi))])
    out["vol"] = ([K[c][:, :Bv] for c in range(3)], [list(range(Bv))])
    for i in range(4):
        out[f"tr{i}"] = ([R[i].T], [c for c in (list(range(irows)), list(range(irows, B))) if c])
    # the four lifts accumulate into the same registers: shared output groups, one input
    # partition per face
    out["lift"] = ([R[i] for i in range(4)], [list(range(Bt))], [0, 1, 2, 3])
    return out


def _chunks(rows, s):
    return [rows[i:i + s] for i in range(0, len(rows), s)]


class _Problem:
    def __init__(self, mats, nin, part_of):
        self.mats = [m.astype(np.int32) for m in mats]
        self.nin = nin
        self.part_of = part_of  # input partition used by each matrix

    def cost(self, og, igs):
        Gs = []
        for ig in igs:
            G = np.zeros((self.nin, len(ig)), np.int32)
            for j, g in enumerate(ig):
                G[g, j] = 1
            Gs.append(G)
        c = 0
        for m, pi in zip(self.mats, self.part_of):
            rows = np.stack([m[g].any(axis=0) for g in og]).astype(np.int32)  # (n_og, nin)
            c += int(((rows @ Gs[pi]) > 0).sum())
        return c


def anneal(mats, classes, part_of=None, iters=20000, seed=0, restarts=3):
    """Partition the output rows (groups of 8) and, per input partition, the input rows
    (groups of 4, never mixing two classes) to minimise the nonzero-tile count."""
    nout, nin = mats[0].shape
    part_of = part_of or [0] * len(mats)
    nparts = max(part_of) + 1
    prob = _Problem(mats, nin, part_of)
    cls_of = []
    for ci, cl in enumerate(classes):
        cls_of += [ci] * len(_chunks(list(cl), 4))
    best = None
    for r in range(restarts):
        rng = random.Random(seed * 1000 + r)
        og = _chunks(list(range(nout)), 8)
        igs = [[g for cl in classes for g in _chunks(list(cl), 4)] for _ in range(nparts)]
        if r > 0:  # random start
            perm = list(range(nout))
            rng.shuffle(perm)
            og = _chunks(perm, 8)
            for k in range(nparts):
                igs[k] = []
                for cl in classes:
                    cl = list(cl)
                    rng.shuffle(cl)
                    igs[k] += _chunks(cl, 4)
        cur = prob.cost(og, igs)
        bc, bo_, bi_ = cur, [g[:] for g in og], [[g[:] for g in ig] for ig in igs]
        T = 1.5
        for it in range(iters):
            k = rng.randrange(nparts + 1)
            G = og if k == nparts else igs[k]
            if len(G) < 2:
                continue
            a, b = rng.sample(range(len(G)), 2)
            if G is not og and cls_of[a] != cls_of[b]:
                continue
            i = rng.randrange(len(G[a]))
            j = rng.randrange(len(G[b]))
            G[a][i], G[b][j] = G[b][j], G[a][i]
            c = prob.cost(og, igs)
            if c <= cur or rng.random() < math.exp((cur - c) / T):
                cur = c
                if c < bc:
                    bc, bo_, bi_ = c, [g[:] for g in og], [[g[:] for g in ig] for ig in igs]
            else:
                G[a][i], G[b][j] = G[b][j], G[a][i]
            T = max(0.05, T * 0.9997)
        if best is None or bc < best[0]:
            best = (bc, bo_, bi_)
    bc, og, igs = best
    return {"tiles": bc, "out": [sorted(g) for g in og], "in": [[sorted(g) for g in ig] for ig in igs]}


def _path(N):
    return os.path.join(CACHE_DIR, f"N{N}.json")


def tiling(N):
    """Cached groupings for order N: {product: {"tiles", "out", "in"}}."""
    if not os.path.exists(_path(N)):
        raise KeyError(f"no cached tiling for N={N}; run python -m paper_1903_11521_b200.gen.tiling --search {N}")
    with open(_path(N)) as fh:
        return json.load(fh)


def _store(N, res):
    os.makedirs(CACHE_DIR, exist_ok=True)
    with open(_path(N), "w") as fh:
        json.dump(res, fh, separators=(",", ":"))


def search(N, iters=20000):
    res = {}
    for name, pr in products(N).items():
        res[name] = anneal(*pr, iters=iters)
        print(f"N={N} {name}: {res[name]['tiles']} tiles", flush=True)
    _store(N, res)
    return res


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--search":
        for n in args[1:]:
            search(int(n))
    elif args and args[0] == "--redo":  # --redo PREFIX N...: re-search the products starting with PREFIX
        pre = args[1]
        for n in args[2:]:
            res = tiling(int(n))
            for name, pr in products(int(n)).items():
                if name.startswith(pre):
                    res[name] = anneal(*pr)
                    print(f"N={n} {name}: {res[name]['tiles']} tiles", flush=True)
            _store(int(n), res)
