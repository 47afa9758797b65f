"""Generator of the FP64 tensor-core (DMMA m8n8k4) form of the global-matrix products.

Every product of a global matrix with a tile of 32 elements x 9 quantity columns,

    CK        D^{d+1} (+)= Ktilde^c[:B_{d+1}, :B_d]  (D^d A*^cT)
    volume    Q      +=  Khat^c[:, :Bv]            (I A*^cT)
    trace     T_i     =  R^iT                       I
    lift      Q      +=  R^i                        Y_i

is a GEMM with M = matrix rows, K = matrix columns and N = 288 data columns, issued as
8x4 matrix tiles (the DMMA A operand).  The rows of a tile are not fixed blocks: an
m-tile is any 8 output rows and a k-set any 4 input rows (gen/tiling.py chooses them to
minimise the number of nonzero tiles -- the zero-block exploitation of the paper's
equivalent sparsity patterns, with free block boundaries).  Input rows reach
the B operand either through the warp-private star chunk X (CK, volume: the chunk is
built from the 4 rows named at compile time) or by a per-lane gathered shared-memory load
(trace, lift: lane row = byte (lane & 3) of a 32-bit immediate); accumulator rows are
scattered on write-back (row = byte (lane >> 2) of a 64-bit immediate, 0xff = padding).

Each of the 12 warps owns three 8-column data tiles (quantities 3g..3g+2, elements
8ct..8ct+7), so every B operand it feeds to a DMMA is warp-private.  A fragments are
stored lane-ordered (lane i holds A[i/4][i%4]) in a device table, one coalesced 256-byte
load per tile, issued one k-set ahead of use.

Emits ``csrc/generated/ydg_dmma_N{n}.cuh``.
"""
from __future__ import annotations

import os

from . import einsum, tables, tiling

ORDERS = (1, 2, 3, 4, 5, 6)
PAD = 0xFF


def r8(x):
    return (x + 7) // 8 * 8


class Table:
    def __init__(self):
        self.frags = []  # list of 32-value lists

    def add(self, M, rows, cols):
        """Fragment of matrix M (callable (row, col) -> value) on the given output rows (8,
        None = padding) and input columns (4, None = padding); None if all zero."""
        vals = []
        for i in range(32):
            r, c = rows[i // 4], cols[i % 4]
            vals.append(0.0 if r is None or c is None else float(M(r, c)))
        if not any(v != 0.0 for v in vals):
            return None
        self.frags.append(vals)
        return len(self.frags) - 1


class Pool:
    """fp64 coefficients of the sparse DFMA code, placed in a __constant__ array so that each
    DFMA reads its coefficient as a constant-bank operand (a literal would cost two uniform
    register moves per DFMA: there are no 64-bit immediates)."""

    def __init__(self, name):
        self.name = name
        self.vals = []
        self.index = {}

    def __call__(self, v):
        v = float(v)
        if v not in self.index:
            self.index[v] = len(self.vals)
            self.vals.append(v)
        return f"{self.name}[{self.index[v]}]"


POOL = None


def lit(v):
    return POOL(v) if POOL is not None else repr(float(v))


def pad_rows(g, n):
    return list(g) + [None] * (n - len(g))


def row_word64(rows):
    w = 0
    for i, r in enumerate(pad_rows(rows, 8)):
        w |= (PAD if r is None else r) << (8 * i)
    return f"0x{w:016x}ULL"


def kset_word(rows):
    """32-bit gather word; padding slots repeat the first row (their A column is zero)."""
    rr = list(rows) + [rows[0]] * (4 - len(rows))
    w = 0
    for i, r in enumerate(rr):
        w |= r << (8 * i)
    return f"0x{w:08x}u"


def kset_rows(rows):
    return list(rows) + [rows[0]] * (4 - len(rows))


class Emit:
    def __init__(self):
        self.lines = []
        self.n = 0

    def __call__(self, s):
        self.lines.append(s)


def afrag_expr(tid, fbase, kind="l"):
    """A-fragment load: products that may be staged in shared memory (fbase = first table
    index staged; kind l = local kernel, f = flux kernel) or the global table (L1-cached)."""
    return f"afrag(x, {tid})" if fbase is None else f"afrag_{kind}(x, {tid}, {tid - fbase})"


def plan_xprod(tab, mats, til):
    plan = []  # per k-set: list of (c, mt, tid)
    for ks in til["in"][0]:
        cols = pad_rows(ks, 4)
        tiles = []
        for c, M in enumerate(mats):
            for mt, og in enumerate(til["out"]):
                tid = tab.add(M, pad_rows(og, 8), cols)
                if tid is not None:
                    tiles.append((c, mt, tid))
        plan.append(tiles)
    return plan


def emit_xprod(b, plan, name, til, src, fbase=None, acc="acc", pipe=False):
    """CK / volume style product: per k-set the warp-private star chunk X^c of the 4 rows
    (uniform across lanes), then per c the DMMAs of that c's nonzero tiles.  A fragments of
    the next k-set are loaded before the current k-set's work.  pipe: software-pipelined
    (the chunk of k-set i + 1 computed beside k-set i's DMMAs, two buffers x.xb / x.xb2)."""
    ins = til["in"][0]
    b(f"    // {name}: {sum(len(t) for t in plan)} tiles, {len(ins)} k-sets, {len(til['out'])} m-tiles")
    names = [[f"a{i}_{j}" for j in range(len(t))] for i, t in enumerate(plan)]

    def afr(i):
        if plan[i]:
            b("    const double " + ", ".join(f"{nm} = {afrag_expr(t[2], fbase)}" for nm, t in zip(names[i], plan[i])) + ";")

    afr(0)
    if pipe:
        buf = lambda i: "x.xb2" if i & 1 else "x.xb"
        b("    static_assert((B - IROWS) * kRS + kW * kXW <= SROWS * kRS, \"second star-chunk buffer in S\");")
        r = kset_rows(ins[0])
        b(f"    xcalc_to<{src}, B>(x, {buf(0)}, {r[0]}, {r[1]}, {r[2]}, {r[3]});")
        b("    __syncwarp();")
        for i, ks in enumerate(ins):
            if i + 1 < len(ins):
                afr(i + 1)
                r = kset_rows(ins[i + 1])
                b(f"    xcalc_to<{src}, B>(x, {buf(i + 1)}, {r[0]}, {r[1]}, {r[2]}, {r[3]});")
            for c in range(3):
                mine = [(mt, nm) for (cc, mt, tid), nm in zip(plan[i], names[i]) if cc == c]
                if not mine:
                    continue
                b(f"    {{ double bf[kU]; xb_from({buf(i)}, x, {c}, bf);")
                for mt, nm in mine:
                    b(f"      dmma3({acc}[{mt}], {nm}, bf);")
                b("    }")
            b("    __syncwarp();")
        return sum(len(t) for t in plan)
    for i, ks in enumerate(ins):
        if i + 1 < len(ins):
            afr(i + 1)
        r = kset_rows(ks)
        b(f"    xcalc<{src}, B>(x, {i}, {r[0]}, {r[1]}, {r[2]}, {r[3]});")
        b("    __syncwarp();")
        for c in range(3):
            mine = [(mt, nm) for (cc, mt, tid), nm in zip(plan[i], names[i]) if cc == c]
            if not mine:
                continue
            b(f"    {{ double bf[kU]; xb_b(x, {i}, {c}, bf);")
            for mt, nm in mine:
                b(f"      dmma3({acc}[{mt}], {nm}, bf);")
            b("    }")
    return sum(len(t) for t in plan)


def emit_gprod(b, tab, M, outs, ins, loader, acc="acc", fbase=None):
    """Trace / lift style product: B fragments gathered per lane from memory
    (``loader(kset_index, word)`` returns the C expression filling ``bf``)."""
    plan = []
    for ks in ins:
        cols = pad_rows(ks, 4)
        tiles = []
        for mt, og in enumerate(outs):
            tid = tab.add(M, pad_rows(og, 8), cols)
            if tid is not None:
                tiles.append((mt, tid))
        plan.append(tiles)
    n = 0
    live = [(i, ks, t) for i, (ks, t) in enumerate(zip(ins, plan)) if t]
    names = {i: [f"g{i}_{j}" for j in range(len(t))] for i, _, t in live}
    if live:
        i0 = live[0][0]
        b("      const double " + ", ".join(f"{nm} = {afrag_expr(t[1], fbase, 'f')}" for nm, t in zip(names[i0], live[0][2])) + ";")
    for k, (i, ks, tiles) in enumerate(live):
        if k + 1 < len(live):
            i1 = live[k + 1][0]
            b("      const double " + ", ".join(f"{nm} = {afrag_expr(t[1], fbase, 'f')}" for nm, t in zip(names[i1], live[k + 1][2])) + ";")
        src = loader(i, kset_word(ks))
        b(f"      {{ {src}")
        for (mt, tid), nm in zip(tiles, names[i]):
            b(f"        dmma3({acc}[{mt}], {nm}, bf);")
        b("      }")
        n += len(tiles)
    return n


# CK steps with at most this many output rows run as sparse DFMA code (CTA-wide)
DFMA_CK_ROWS = int(os.environ.get("YDG_GEN_CKROWS", "20"))
# faces 0 and 1 traces as sparse DFMA code (else tensor cores); faces 2 and 3 as well
DFMA_TR01 = os.environ.get("YDG_GEN_TR01", "1") == "1"
DFMA_TR23 = os.environ.get("YDG_GEN_TR23", "0") == "1"
# CK step 0's star chunks software-pipelined against the previous k-set's DMMAs
XPIPE = os.environ.get("YDG_GEN_XPIPE", "0") == "1"
# where the sparse-DFMA CK steps load the column's star coefficients: "step" (each step,
# from global memory), "tail" (once, after CK step 0), "pre" (once, before CK step 0)
STAR_LOAD = os.environ.get("YDG_GEN_STAR", "step")
DFMA_TAIL_ROWS = 0   # CK steps d >= 1 from the first with at most this many output rows on:
                     # one warp-synchronous sparse DFMA phase (0 = off: the element-grouped
                     # lanes hit 9-way shared-memory bank conflicts, measured slower)


def emit_ck_dfma(b, d, K, bi, bo, IROWS):
    """Small CK step as constant-coefficient DFMAs, one thread per data column (element ce,
    quantity cp): y_k = sum_c sum_l Ktilde^c[k][l] X^c[l], X^c = D A*^cT of the column, only
    the nonzeros of Ktilde (exact nonzero count; no 8x4 tile padding)."""
    nz = {}
    n = 0
    for c in range(3):
        for k in range(bo):
            for l in range(bi):
                v = -K[c][l][k]
                if v != 0.0:
                    nz.setdefault(l, []).append((c, k, v))
                    n += 1
    src = "SRC_Q" if d == 0 else "SRC_S"
    b(f"  // CK step d = {d}: rows in {bi}, rows out {bo}; sparse DFMA ({n} nonzeros)")
    own_star = STAR_LOAD == "step" or d == 0
    if own_star:
        b(f"  static __device__ __forceinline__ void ck{d}(Ctx& x) {{")
    else:
        b(f"  static __device__ __forceinline__ void ck{d}(Ctx& x, const double (&ca)[9], int q0, int q1, int q2) {{")
    b(f"    double y[{bo}];")
    b(f"    for (int k = 0; k < {bo}; ++k) y[k] = 0.0;")
    b("    if (x.cc < kRS) {")
    if own_star:
        b("      double ca[9];")
        b("      int q0, q1, q2;")
        b("      col_star(x, x.ce, x.cp, ca, q0, q1, q2);")
    for l in sorted(nz):
        b(f"      {{ double x0, x1, x2; col_x<{src}, B>(x, {l}, x.ce, ca, q0, q1, q2, x0, x1, x2);")
        for c, k, v in nz[l]:
            b(f"        y[{k}] = fma({lit(v)}, x{c}, y[{k}]);")
        b("      }")
    b("    }")
    b("    x.sync();  // every read of D^d done")
    b(f"    if (x.cc < kRS) col_wb<{1 if d == 0 else 0}, {bo}>(x, x.cc, y, {d});")
    if d == 0 and IROWS > bo:
        b(f"    scale_irows<{bo}, {IROWS}>(x);  // rows of I fed by D^0 only: dt * Q")
    b("    x.sync();")
    b("  }")
    return -n  # negative: nonzero FMAs (not tiles)


def emit_ck_tail(b, d0, N, K):
    """CK steps d0..N-1 (few output rows) as one warp-synchronous phase of constant-
    coefficient DFMAs: thread (element te, quantity tp) -- the 9 quantities of an element
    sit in one warp (3 elements per warp), so the cross-quantity star products need only
    __syncwarp between steps, no CTA barrier.  Nonzeros of Ktilde only."""
    n = 0
    b(f"  // CK steps {d0}..{N - 1}: warp-synchronous sparse DFMA tail")
    b("  static __device__ __forceinline__ void ck_tail(Ctx& x) {")
    b("    double ca[9];")
    b("    int q0 = 0, q1 = 0, q2 = 0;")
    b("    if (x.tc >= 0) col_star(x, x.te, x.tp, ca, q0, q1, q2);")
    for d in range(d0, N):
        bi, bo = einsum.ck_dims(N, d)
        nz = {}
        for c in range(3):
            for k in range(bo):
                for l in range(bi):
                    v = -K[c][l][k]
                    if v != 0.0:
                        nz.setdefault(l, []).append((c, k, v))
                        n += 1
        b(f"    {{  // step d = {d}: rows in {bi}, rows out {bo}")
        b(f"      double y[{bo}];")
        b(f"      for (int k = 0; k < {bo}; ++k) y[k] = 0.0;")
        b("      if (x.tc >= 0) {")
        for l in sorted(nz):
            b(f"        {{ double x0, x1, x2; col_x<SRC_S, B>(x, {l}, x.te, ca, q0, q1, q2, x0, x1, x2);")
            for c, k, v in nz[l]:
                b(f"          y[{k}] = fma({lit(v)}, x{c}, y[{k}]);")
            b("        }")
        b("      }")
        b("      __syncwarp();  // every read of the element's D^d done")
        b(f"      if (x.tc >= 0) col_wb<0, {bo}>(x, x.tc, y, {d});")
        b("      __syncwarp();")
        b("    }")
    b("    x.sync();  // the time integral is complete")
    b("  }")
    return -n


def emit_trace01_dfma(b, R, B, Bt, IROWS, TS, faces=(0, 1), fname="trace01"):
    """Traces of two faces (the two sparsest, 0 and 1, by default) as constant-coefficient
    DFMAs, one thread per data column: T_F[m] = sum_k R^F[k][m] I[k] over the nonzeros, both
    faces from one pass over the column; results go to the two staging blocks [lane][m][q]."""
    n = 0
    fa, fb = faces
    b(f"  // traces of faces {fa} and {fb} (sparse DFMA, one thread per data column)")
    b(f"  static __device__ __forceinline__ void {fname}(Ctx& x, double* stg0, double* stg1) {{")
    b("    if (x.cc >= kRS) return;")
    b(f"    double t0[{Bt}], t1[{Bt}];")
    b(f"    for (int m = 0; m < {Bt}; ++m) t0[m] = t1[m] = 0.0;")
    gk = [k for k in range(IROWS, B) if any(R[F][k][m] != 0.0 for F in faces for m in range(Bt))]
    if gk:  # rows >= IROWS (dt * Q, global memory): all loads first, latency under the smem rows
        b(f"    double qg[{len(gk)}];")
        for i, k in enumerate(gk):
            b(f"    qg[{i}] = ld_stream(x.Qt + {k} * kRS + x.cc);")
    for k in list(range(IROWS)) + gk:
        terms = [(j, m, R[F][k][m]) for j, F in enumerate(faces) for m in range(Bt) if R[F][k][m] != 0.0]
        if not terms:
            continue
        src = f"x.I[swz({k}, x.cc)]" if k < IROWS else f"x.dt * qg[{gk.index(k)}]"
        b(f"    {{ const double ik = {src};")
        for j, m, v in terms:
            b(f"      t{j}[{m}] = fma({lit(v)}, ik, t{j}[{m}]);")
            n += 1
        b("    }")
    b(f"    for (int m = 0; m < {Bt}; ++m) {{")
    b(f"      stg0[x.ce * {TS} + m * kP + x.cp] = t0[m];")
    b(f"      stg1[x.ce * {TS} + m * kP + x.cp] = t1[m];")
    b("    }")
    b("  }")
    return n


def gen_order(N):
    global POOL
    POOL = Pool(f"cdf_N{N}")
    t = tables.load(N)
    K, R, f = tables.kdir(t), t["R"], t["f"]  # CK / volume in the sparser directions (tables.KDIR_T)
    B, Bt = t["B"], t["Bt"]
    Bv = einsum.vol_dim(N)
    til = tiling.tiling(N)
    tab = Table()
    IROWS = Bv  # time-integral rows in shared memory (rows >= Bv are dt * Q)
    SROWS = Bv  # rows of D^d, d >= 1
    TS = (9 * Bt + 1) // 2 * 2
    QMT = len(til["vol"]["out"])
    LMT = len(til["lift"]["out"])
    TMT = max(len(til[f"tr{i}"]["out"]) for i in range(4))
    body = []
    b = body.append
    counts = {}
    tail0 = None
    regions = {}  # products whose A fragments are staged in shared memory: [first, end)
    # ---------------- CK
    for d in range(N):
        bi, bo = einsum.ck_dims(N, d)
        tl = til[f"ck{d}"]
        MT = len(tl["out"])
        mats = [(lambda r, col, c=c: -K[c][col][r]) for c in range(3)]  # Kt^c[r][col] = -K^c[col][r]
        if d >= 1 and bo <= DFMA_TAIL_ROWS:
            tail0 = d
            counts["ck_tail"] = emit_ck_tail(b, d, N, K)
            break
        if bo <= DFMA_CK_ROWS:
            counts[f"ck{d}"] = emit_ck_dfma(b, d, K, bi, bo, IROWS)
            continue
        b(f"  // CK step d = {d}: rows in {bi}, rows out {bo}")
        b(f"  static __device__ __forceinline__ void ck{d}(Ctx& x) {{")
        b(f"    double acc[{MT}][kU][2];")
        b("    zero_acc(acc);")
        f0 = len(tab.frags)
        plan = plan_xprod(tab, mats, tl)
        if d == 0:  # staged in the shared-memory fragment buffer
            regions["CK0"] = (f0, len(tab.frags))
        counts[f"ck{d}"] = emit_xprod(b, plan, f"ck{d}", tl, "SRC_Q" if d == 0 else "SRC_S",
                                      fbase=f0 if d == 0 else None, pipe=d == 0 and XPIPE)
        b("    x.sync();  // every read of D^d done")
        for mt, og in enumerate(tl["out"]):
            b(f"    ck_wb<{1 if d == 0 else 0}, B>(x, acc[{mt}], {d}, {row_word64(og)});")
        if d == 0 and IROWS > bo:
            b(f"    scale_irows<{bo}, {IROWS}>(x);  // rows of I fed by D^0 only: dt * Q")
        b("    x.sync();")
        b("  }")
    b("  static __device__ __forceinline__ void ck(Ctx& x) {")
    dfma_steps = [d for d in range(1, tail0 if tail0 is not None else N) if einsum.ck_dims(N, d)[1] <= DFMA_CK_ROWS]
    star_args = ""
    if STAR_LOAD != "step" and dfma_steps:
        star_args = ", ca, q0, q1, q2"
        b("    double ca[9];")
        b("    int q0 = 0, q1 = 0, q2 = 0;")
    for d in range(tail0 if tail0 is not None else N):
        if star_args and ((STAR_LOAD == "pre" and d == 0) or (STAR_LOAD == "tail" and d == dfma_steps[0])):
            b("    if (x.cc < kRS) col_star(x, x.ce, x.cp, ca, q0, q1, q2);")
        b(f"    ck{d}(x{star_args if d in dfma_steps else ''});")
        if d == 0:
            b("    after_ck0<" + str(N) + ">(x);  // the fragment buffer is free: stage the volume's")
        b(f"    YDG_PHASE({2 + d});")
    if tail0 is not None:
        b("    ck_tail(x);")
        b(f"    YDG_PHASE({2 + tail0});")
    b("  }")
    # ---------------- volume
    tl = til["vol"]
    mats = [(lambda r, col, c=c: K[c][r][col]) for c in range(3)]
    b(f"  // volume: Q += sum_c Khat^c (I A*^cT)")
    b(f"  static __device__ __forceinline__ void volume(Ctx& x, double (&acc)[{QMT}][kU][2]) {{")
    f0 = len(tab.frags)
    plan = plan_xprod(tab, mats, tl)
    regions["VOL"] = (f0, len(tab.frags))
    counts["vol"] = emit_xprod(b, plan, "vol", tl, "SRC_I", fbase=f0)
    b("  }")
    b(f"  static __device__ __forceinline__ void add_volume(const Ctx& x, double* Qt, double (&acc)[{QMT}][kU][2], const double* Qs,")
    b("                                                   const double2 (*pre)[kU] = nullptr) {")
    b("    constexpr unsigned long long w[] = {" + ", ".join(row_word64(og) for og in tl["out"]) + "};")
    b("    add_q<" + str(QMT) + ", IROWS>(x, Qt, acc, w, Qs, pre);")
    b("  }")
    b("  // the first batch's Q rows >= IROWS (global memory), loaded ahead of the volume product")
    b("  static __device__ __forceinline__ void add_volume_pre(const Ctx& x, const double* Qt, double2 (&v)[2][kU]) {")
    b("    constexpr unsigned long long w[] = {" + ", ".join(row_word64(og) for og in tl["out"]) + "};")
    b("    q_pre<" + str(QMT) + ", IROWS>(x, Qt, w, v);")
    b("  }")
    # ---------------- traces T_i = R^iT I
    counts["tr01_dfma"] = emit_trace01_dfma(b, R, B, Bt, IROWS, TS) if DFMA_TR01 else 0
    counts["tr23_dfma"] = emit_trace01_dfma(b, R, B, Bt, IROWS, TS, (2, 3), "trace23") if DFMA_TR01 and DFMA_TR23 else 0
    b(f"  static constexpr bool TR01_DFMA = {'true' if DFMA_TR01 else 'false'};")
    b(f"  static constexpr bool TR23_DFMA = {'true' if DFMA_TR01 and DFMA_TR23 else 'false'};")
    b(f"  // trace: T_F = R^FT I (rows < IROWS of I from shared memory, dt * Q from global memory);")
    b(f"  // the C fragments go to the staging block [lane][m][q] (stride TS)")
    b(f"  template <int F> static __device__ __forceinline__ void trace(Ctx& x, double* stg) {{")
    for i in range(4):
        tl = til[f"tr{i}"]
        ins = tl["in"][0]
        outs = tl["out"]
        b(f"    {'if' if i == 0 else 'else if'} constexpr (F == {i}) {{")
        b(f"      double acc[{len(outs)}][kU][2];")
        b("      zero_acc(acc);")
        gl = [k for k, ks in enumerate(ins) if ks[0] >= IROWS]
        if gl:
            b(f"      double bq[{len(gl)}][kU];  // global B fragments first (latency overlap)")
            for n_, k in enumerate(gl):
                b(f"      gq_b<B>(x, {kset_word(ins[k])}, bq[{n_}]);")

        def loader(k, w, gl=gl):
            if k in gl:
                return f"const double (&bf)[kU] = bq[{gl.index(k)}];"
            return f"double bf[kU]; ismem_b(x, {w}, bf);"
        Mi = lambda r, col, i=i: R[i][col][r]
        counts[f"tr{i}"] = emit_gprod(b, tab, Mi, outs, ins, loader)
        for mt, og in enumerate(outs):
            b(f"      stage_trace<{TS}>(x, stg, acc[{mt}], {row_word64(og)});")
        b("    }")
    b("  }")
    # ---------------- lift Q += R^i Y_i: m-tile-group major (two m-tiles at a time), the Q
    # rows of the next group loaded while the current group's DMMAs run
    tl = til["lift"]
    outs = tl["out"]
    groups = [list(range(g, min(g + 2, len(outs)))) for g in range(0, len(outs), 2)]
    counts["lift"] = 0
    lift0 = len(tab.frags)
    # paired lift: faces 2P and 2P+1 accumulate into the same registers, one Q update per pair
    b(f"  // paired lift + Q update (flux kernel layout): Q += R^(2P) Ya + R^(2P+1) Yb")
    # lift2_pre: the first m-tile group's Q rows, issued by the caller ahead of the lift
    g0 = groups[0]
    b(f"  static __device__ __forceinline__ void lift2_pre(const Ctx& x, const double* Qt, double2 (&qn)[2][kU]) {{")
    b(f"    load_qf(x, Qt, {row_word64(outs[g0[0]])}, {row_word64(outs[g0[1]]) if len(g0) > 1 else '~0ULL'}, qn);")
    b("  }")
    b(f"  template <int P> static __device__ __forceinline__ void lift2(Ctx& x, const double* Ya, const double* Yb, double* Qt, double2 (&qn)[2][kU]) {{")
    for P in range(2):
        b(f"    {'if' if P == 0 else 'else if'} constexpr (P == {P}) {{")
        for gi, grp in enumerate(groups):
            b("      {")
            b("        double2 qc[2][kU];")
            b("        copy_q2(qn, qc);")
            if gi + 1 < len(groups):
                g1 = groups[gi + 1]
                b(f"        load_qf(x, Qt, {row_word64(outs[g1[0]])}, {row_word64(outs[g1[1]]) if len(g1) > 1 else '~0ULL'}, qn);")
            b("        double acc[2][kU][2];")
            b("        zero_acc(acc);")
            sub = [outs[m] for m in grp]
            for i, yv in ((2 * P, "Ya"), (2 * P + 1, "Yb")):
                Mi = lambda r, col, i=i: R[i][r][col]
                b("        {")
                counts["lift"] += emit_gprod(b, tab, Mi, sub, tl["in"][i],
                                             lambda k, w, yv=yv: f"double bf[kU]; smem_bf(x, {yv}, {w}, bf);", fbase=lift0)
                b("        }")
            b(f"        store_qf(x, Qt, {row_word64(outs[grp[0]])}, {row_word64(outs[grp[1]]) if len(grp) > 1 else '~0ULL'}, acc, qc);")
            b("      }")
        b("    }")
    b("  }")
    regions["LIFT"] = (lift0, len(tab.frags))
    regions.setdefault("CK0", (0, 0))  # CK step 0 ran as sparse DFMA code
    # ---------------- neighbour orientation z = f^h t, uniform over lanes:
    # f^1 = S (diagonal +-1) and f^2 = S f^0 S, so t' = (h != 0 ? S t : t), u = f^0 t',
    # z = (h == 1 ? t' : (h == 2 ? S u : u))
    S = [f[1][m][m] for m in range(Bt)]
    for m in range(Bt):
        for n in range(Bt):
            assert (m == n) or f[1][m][n] == 0.0
            assert abs(f[2][m][n] - S[m] * f[0][m][n] * S[n]) < 1e-14
    b("  // z = f^h t (P:1342) for every lane's own h, without divergence (f^1 = S diagonal,")
    b("  // f^2 = S f^0 S); row m goes to Y[m][col] (swizzled rows of the flux staging)")
    b(f"  static __device__ __forceinline__ void rotf(int h, double (&t)[{Bt}], double* Y, int col) {{")
    b("    const bool fl = h != 0, id = h == 1, s2 = h == 2;")
    for n in range(Bt):
        if S[n] < 0:
            b(f"    t[{n}] = fl ? -t[{n}] : t[{n}];")
    for m in range(Bt):
        terms = [(n, f[0][m][n]) for n in range(Bt) if f[0][m][n] != 0.0]
        expr = None
        for n, v in terms:
            # literals here: the flux kernel's register budget (constant-bank operands spilled)
            expr = f"{float(v)!r} * t[{n}]" if expr is None else f"fma({float(v)!r}, t[{n}], {expr})"
        b(f"    {{ const double u = {expr or '0.0'};")
        if S[m] < 0:
            b(f"      Y[swzf({m}, col)] = id ? t[{m}] : (s2 ? -u : u); }}")
        else:
            b(f"      Y[swzf({m}, col)] = id ? t[{m}] : u; }}")
    b("  }")
    pool = POOL.vals or [0.0]
    cdecl = [f"// coefficients of the sparse DFMA code (constant-bank operands)",
             f"__constant__ double cdf_N{N}[{len(pool)}] = {{"]
    for s0 in range(0, len(pool), 6):
        cdecl.append("  " + ", ".join(repr(v) for v in pool[s0:s0 + 6]) + ",")
    cdecl.append("};")
    lines = [f"// GENERATED by paper_1903_11521_b200/gen/dmma.py for N = {N} -- do not edit.",
             "#pragma once", "namespace ydg {", "namespace dm {"] + cdecl + [f"template <> struct DG<{N}> {{",
             f"  static constexpr int N = {N}, B = {B}, Bt = {Bt}, Bv = {Bv};",
             f"  static constexpr int SROWS = {SROWS};  // rows of S (D^d, d >= 1)",
             f"  static constexpr int IROWS = {IROWS};  // rows of the time-integral region",
             f"  static constexpr int TS = {TS};  // doubles per element-face trace block [m][q]",
             f"  static constexpr int QMT = {QMT}, LMT = {LMT}, TMT = {TMT};",
             f"  static constexpr int NFRAG = {len(tab.frags)};",
             "  // A-fragment ranges staged in shared memory (first, count)",
             f"  static constexpr int CK0_F0 = {regions['CK0'][0]}, CK0_NF = {regions['CK0'][1] - regions['CK0'][0]};",
             f"  static constexpr int VOL_F0 = {regions['VOL'][0]}, VOL_NF = {regions['VOL'][1] - regions['VOL'][0]};",
             f"  static constexpr int LIFT_F0 = {regions['LIFT'][0]}, LIFT_NF = {regions['LIFT'][1] - regions['LIFT'][0]};",
             "  // DMMA tiles per product (x 4 col tiles x 9 warps per 32-element tile): " +
             ", ".join(f"{k} {v}" for k, v in counts.items())]
    lines += body
    lines.append("};")
    lines.append(f"__device__ const double frag_N{N}[{max(1, len(tab.frags)) * 32}] = {{")
    flat = [v for fr in tab.frags for v in fr] or [0.0] * 32
    for s in range(0, len(flat), 8):
        lines.append("  " + ", ".join(repr(float(v)) if v != 0 else "0.0" for v in flat[s:s + 8]) + ",")
    lines.append("};")
    lines.append(f"template <> __device__ __forceinline__ const double* frag_table<{N}>() {{ return frag_N{N}; }}")
    # dense neighbour-orientation matrices f^h, h = 0..2 (block-diagonal by face degree)
    lines.append(f"__device__ const double fh_N{N}[{3 * Bt * Bt}] = {{")
    flat = [float(f[h][m][n]) for h in range(3) for m in range(Bt) for n in range(Bt)]
    for s0 in range(0, len(flat), 8):
        lines.append("  " + ", ".join(repr(v) if v != 0 else "0.0" for v in flat[s0:s0 + 8]) + ",")
    lines.append("};")
    lines.append(f"template <> __device__ __forceinline__ const double* fh_table<{N}>() {{ return fh_N{N}; }}")
    lines.append("}  // namespace dm")
    lines.append("}  // namespace ydg")
    return "\n".join(lines) + "\n", counts


def dmma_counts(N):
    """(tensor-core MACs executed per element) of the DMMA products."""
    til = tiling.tiling(N)
    n = sum(v["tiles"] for v in til.values())
    return n * 32 * 9


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    outdir = os.path.join(here, "..", "csrc", "generated")
    for N in ORDERS:
        text, counts = gen_order(N)
        with open(os.path.join(outdir, f"ydg_dmma_N{N}.cuh"), "w") as fh:
            fh.write(text)
        print(f"N={N}: {counts}")


if __name__ == "__main__":
    main()
