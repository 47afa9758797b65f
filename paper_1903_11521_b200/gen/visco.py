"""Generator of the viscoelastic (P = 27) FP64 tensor-core local kernel's products.

The viscoelastic CK recursion, volume, traces and lift (
P:1312-1342 with the source term of reading R14) apply the same global matrices as the
elastic scheme to a tile of 8 elements x 27 quantities (216 data columns).  Each product
Y (+)= M X with M in {Ktilde^c, K^c, R^i, R^iT} runs as DMMA m8n8k4 tiles: the 8 output
rows of an m-tile are gathered freely (annealed, gen/tiling.py; the accumulator rows are
scattered on write-back) and the input rows form FIXED consecutive k-sets of 4, so that
the B fragments built from shared memory are bank-conflict free.  Zero 8x4 blocks are
skipped (the zero-block exploitation of P:1351-1374).

Emits ``csrc/generated/ydg_visco.cuh``: per order N <= 4 the row tables, the A-fragment
table and four straight-line product functions (CK step and volume left-first, i.e.
Z^c_t = M^c D_t per elastic quantity t; traces; lift) written
against a small context interface implemented in csrc/visco.cu:

    x.ib(buf, ks)          B fragment of the warp's quantity column of D / I, rows 4ks..4ks+3
    x.mma1(acc, f, buf)    acc += frag f x B1[buf]
    x.mma(acc, f, buf)     acc[u] += frag f x B[buf][u], u = 0..2 (lift)
    x.acoef(i)             flux-solver coefficients of face i (lift)
    x.ychunk(buf, i, ks)   B fragments of Y_i = T_i A+_iT, rows 4ks..4ks+3 of face i

    python -m paper_1903_11521_b200.gen.visco
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import tables, tiling

HERE = os.path.dirname(os.path.abspath(__file__))
ORDERS = (1, 2, 3, 4)
CACHE = os.path.join(HERE, "tilings", "visco.json")


def _nz(m):
    return np.abs(m) > 0


def _ceil(a, b):
    return (a + b - 1) // b


def matrices(N):
    t = tables.load(N)
    K = [np.array(k, dtype=np.float64) for k in tables.kdir(t)]  # sparser directions (tables.KDIR_T)
    R = [np.array(r, dtype=np.float64) for r in t["R"]]
    B, Bt = K[0].shape[0], R[0].shape[1]
    ck = [-k.T for k in K]                                    # Ktilde^c = -K^cT (M = I)
    vol = K                                                   # Khat^c = K^c
    lift = [np.hstack([r, np.zeros((B, B - Bt))]) for r in R]  # R^i padded to B input rows
    tr = [r.T for r in R]                                     # T_i = R^iT I
    return B, Bt, ck, vol, lift, tr


def _fixed_classes(nin):
    return [list(range(i, min(i + 4, nin))) for i in range(0, nin, 4)]


def _search(N, iters=8000):
    B, Bt, ck, vol, lift, tr = matrices(N)
    out = {}
    for name, mats in (("ck", ck), ("q", vol + lift), ("tr", tr)):
        nin = mats[0].shape[1]
        res = tiling.anneal([_nz(m) for m in mats], _fixed_classes(nin), iters=iters, restarts=3)
        out[name] = res["out"]
    return out


def partitions(N, redo=False):
    data = {}
    if os.path.exists(CACHE):
        with open(CACHE) as fh:
            data = json.load(fh)
    if redo or str(N) not in data:
        data[str(N)] = _search(N)
        with open(CACHE, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
    return data[str(N)]


class Frags:
    def __init__(self):
        self.vals = []
        self.index = {}

    def add(self, M, rows, ks):
        fr = []
        for lane in range(32):
            r = rows[lane // 4] if lane // 4 < len(rows) else None
            c = 4 * ks + lane % 4
            fr.append(0.0 if r is None or c >= M.shape[1] else float(M[r, c]))
        key = tuple(fr)
        if key not in self.index:
            self.index[key] = len(self.vals)
            self.vals.append(fr)
        return self.index[key]


def _tiles(mats, og, nks):
    """[(ks, [(mat, mt, rows)])] of the nonzero 8x4 blocks, k-set major."""
    res = []
    for ks in range(nks):
        lst = []
        for mi, M in enumerate(mats):
            for mt, rows in enumerate(og):
                blk = M[np.ix_(rows, [c for c in range(4 * ks, 4 * ks + 4) if c < M.shape[1]])]
                if np.any(blk != 0):
                    lst.append((mi, mt, rows))
        res.append((ks, lst))
    return res


def _rowword(rows):
    w = 0
    for i in range(8):
        r = rows[i] if i < len(rows) else 0xFF
        w |= r << (8 * i)
    return w


def gen_order(N):
    B, Bt, ck, vol, lift, tr = matrices(N)
    part = partitions(N)
    fr = Frags()
    L = [f"// ---- order N = {N}: B = {B}, Bt = {Bt}"]
    nks_b, nks_t = _ceil(B, 4), _ceil(Bt, 4)
    counts = {}

    def seq_body(fname, sig, items, first, chunk, mma):
        """items: [(group key, ks, [(mat, mt, frag)])]; software-pipelined one k-set ahead."""
        body = [f"template <class X> __device__ __forceinline__ void {fname}({sig}) {{"]
        items = [it for it in items if it[2]]
        prev_key = None
        for n, (key, ks, lst) in enumerate(items):
            if n == 0:
                body += first(key)
                body.append(f"  {chunk(key, 0, ks)}")
                prev_key = key
            if n + 1 < len(items):
                nk, nks, _ = items[n + 1]
                if nk != prev_key:
                    body += first(nk)
                    prev_key = nk
                body.append(f"  {chunk(nk, (n + 1) & 1, nks)}")
            for (mi, mt, f) in lst:
                body.append(f"  {mma(key, mi, mt, f, n & 1)}")
        body.append("}")
        return body

    # lift first: its fragments take table slots 0..NLIFTF-1 (the neighbour kernel stages
    # only those)
    og = part["q"]
    items = []
    ntile = 0
    for i in range(4):
        for ks, lst in _tiles([lift[i]], og, nks_t):
            items.append((i, ks, [(0, mt, fr.add(lift[i], rows, ks)) for (_, mt, rows) in lst]))
            ntile += len(lst)
    counts["lift"] = ntile
    nliftf = len(fr.vals)
    L += seq_body(f"vlift{N}", f"X& x, double (&a)[{len(og)}][3][2]", items,
                  lambda i: [f"  x.acoef({i});"],
                  lambda i, b, ks: f"x.ychunk({b}, {i}, {ks});",
                  lambda i, mi, mt, f, b: f"x.mma(a[{mt}], {f}, {b});")

    # CK step, left-first: warp t computes Z^c_t = Ktilde^c D_t for c = 0..2 (one B fragment per
    # k-set serves the three directions); the star / source combination follows in shared memory
    og = part["ck"]
    items = []
    ntile = 0
    for ks in range(nks_b):
        lst = []
        for c in range(3):
            for (_, mt, rows) in _tiles([ck[c]], og, nks_b)[ks][1]:
                lst.append((c, mt, fr.add(ck[c], rows, ks)))
        items.append((0, ks, lst))
        ntile += len(lst)
    counts["ck"] = ntile
    L += seq_body(f"vck{N}", f"X& x, double (&a)[3][{len(og)}][2]", items,
                  lambda _: [],
                  lambda _, b, ks: f"x.ib({b}, {ks});",
                  lambda _, c, mt, f, b: f"x.mma1(a[{c}][{mt}], {f}, {b});")
    ck_rows = [_rowword(g) for g in og]

    # volume, left-first (W^c_t = Khat^c I_t), and lift (R^i, chunks of Y_i) share the output rows
    og = part["q"]
    items = []
    ntile = 0
    for ks in range(nks_b):
        lst = []
        for c in range(3):
            for (_, mt, rows) in _tiles([vol[c]], og, nks_b)[ks][1]:
                lst.append((c, mt, fr.add(vol[c], rows, ks)))
        items.append((0, ks, lst))
        ntile += len(lst)
    counts["vol"] = ntile
    L += seq_body(f"vvol{N}", f"X& x, double (&a)[3][{len(og)}][2]", items,
                  lambda _: [],
                  lambda _, b, ks: f"x.ib({b}, {ks});",
                  lambda _, c, mt, f, b: f"x.mma1(a[{c}][{mt}], {f}, {b});")
    q_rows = [_rowword(g) for g in og]

    # traces T_i = R^iT I of one quantity column per warp (all faces per k-set)
    og = part["tr"]
    items = []
    ntile = 0
    for ks, lst in _tiles(tr, og, nks_b):
        items.append((0, ks, [(mi, mt, fr.add(tr[mi], rows, ks)) for (mi, mt, rows) in lst]))
        ntile += len(lst)
    counts["tr"] = ntile
    L += seq_body(f"vtr{N}", f"X& x, double (&t)[4][{len(og)}][2]", items,
                  lambda _: [],
                  lambda _, b, ks: f"x.ib({b}, {ks});",
                  lambda _, mi, mt, f, b: f"x.mma1(t[{mi}][{mt}], {f}, {b});")
    tr_rows = [_rowword(g) for g in og]

    def arr(name, words):
        sel = " : ".join(f"i == {i} ? 0x{w:016x}ull" for i, w in enumerate(words)) + " : ~0ull"
        return f"  __host__ __device__ static constexpr unsigned long long {name}(int i) {{ return {sel}; }}"

    head = [f"template <> struct VT<{N}> {{",
            f"  static constexpr int B = {B}, Bt = {Bt}, BR = {4 * nks_b}, BtR = {4 * nks_t};",
            f"  static constexpr int NCK = {len(ck_rows)}, NQ = {len(q_rows)}, NT = {len(tr_rows)};",
            f"  static constexpr int NFRAG = {len(fr.vals)}, NLIFTF = {nliftf};",
            arr("ck_rows", ck_rows), arr("q_rows", q_rows), arr("tr_rows", tr_rows),
            "};"]
    flat = [v for f in fr.vals for v in f]
    tab = [f"__device__ const double vfrag_N{N}[{len(flat)}] = {{"]
    for s0 in range(0, len(flat), 4):
        tab.append("  " + ", ".join(repr(v) if v != 0 else "0.0" for v in flat[s0:s0 + 4]) + ",")
    tab.append("};")
    tab.append(f"template <> __device__ __forceinline__ const double* vfrag<{N}>() {{ return vfrag_N{N}; }}")
    counts["frags"] = len(fr.vals)
    return head + tab + L, counts


def main():
    out = ["// GENERATED by paper_1903_11521_b200/gen/visco.py -- do not edit.",
           "// Viscoelastic (P = 27) DMMA products: row tables, A fragments, straight-line products.",
           "#pragma once", "namespace ydg { namespace visco {",
           "template <int N> struct VT;", "template <int N> __device__ const double* vfrag();"]
    for N in ORDERS:
        lines, counts = gen_order(N)
        out += lines
        print(f"N={N}: {counts}")
    out.append("}  // namespace visco")
    out.append("}  // namespace ydg")
    path = os.path.join(HERE, "..", "csrc", "generated", "ydg_visco.cuh")
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
