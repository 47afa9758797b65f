"""Host-side checks of the viscoelastic tensor-core kernels' generator and hard-coded patterns
(no GPU).

* gen/visco.py: the tile lists of every product (CK Ktilde^c, volume K^c, lift R^i, traces
  R^iT) rebuild each global matrix exactly from the emitted A fragments -- every nonzero in
  exactly one issued 8x4 tile, every skipped tile zero -- over a partition of the output
  rows into groups of <= 8 and fixed consecutive input k-sets.
* csrc/visco.cu hard-codes the column patterns of the star matrices (non-velocity rows read
  (VU, VV, VW), velocity rows the stress triples) and of the source term; these are pinned
  here against the oracle's own viscoelastic Jacobians and source matrix (oracle/physics.py,
  reading R14), built independently of the library.
* gen/kernels.py: nz_counts_visco counts 51 star nonzeros per direction and 54 source
  nonzeros; pinned against the oracle's matrices.
"""
import numpy as np
import pytest

from oracle import physics
from paper_1903_11521_b200.gen import kernels, visco


def _rebuild(M, og, ks_tiles, nin):
    R = np.zeros(M.shape)
    hits = np.zeros(M.shape, dtype=int)
    for ks, mt, frag in ks_tiles:
        rows = og[mt]
        for lane in range(32):
            if lane // 4 >= len(rows):
                assert frag[lane] == 0.0
                continue
            r, c = rows[lane // 4], 4 * ks + lane % 4
            if c >= nin:
                assert frag[lane] == 0.0
                continue
            R[r, c] += frag[lane]
            hits[r, c] += 1
    return R, hits


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_visco_tiles_rebuild_the_matrices(N):
    B, Bt, ck, vol, lift, tr = visco.matrices(N)
    part = visco.partitions(N)
    for key, mats in (("ck", ck), ("q", vol + lift), ("tr", tr)):
        og = part[key]
        nout, nin = mats[0].shape
        assert sorted(r for g in og for r in g) == list(range(nout)), key
        assert all(len(g) <= 8 for g in og)
        nks = (nin + 3) // 4
        for M in mats:
            fr = visco.Frags()
            tiles = []
            for ks, lst in visco._tiles([M], og, nks):
                for (_, mt, rows) in lst:
                    tiles.append((ks, mt, fr.vals[fr.add(M, rows, ks)]))
            R, hits = _rebuild(M, og, tiles, nin)
            assert np.array_equal(R, M), key
            assert hits.max() <= 1, key
            assert np.all(hits[M != 0] == 1), key
            # a skipped block is a zero block
            issued = {(ks, mt) for ks, mt, _ in tiles}
            for ks in range(nks):
                for mt, rows in enumerate(og):
                    if (ks, mt) not in issued:
                        cols = [c for c in range(4 * ks, 4 * ks + 4) if c < nin]
                        assert not np.any(M[np.ix_(rows, cols)]), key


def _visco_star(seed=3):
    rng = np.random.default_rng(seed)
    rho, vp = 2500.0, 5000.0
    lam, mu = physics.lame(rho, vp, vp / np.sqrt(3.0))
    omega = np.array([0.6, 6.0, 60.0])
    A = physics.jacobians(rho, lam, mu, P=27, omega=omega)
    Jinv = rng.normal(size=(3, 3))  # generic: no accidental zeros
    return physics.star_matrices(Jinv, A), omega


def test_visco_star_pattern_matches_the_kernel():
    """Non-velocity rows of A*^c live on the velocity columns; velocity rows on the stress
    triples (SXX SXY SXZ), (SXY SYY SYZ), (SXZ SYZ SZZ) -- the patterns vm_local hard-codes."""
    star, _ = _visco_star()
    vel_cols = {6: {0, 3, 5}, 7: {3, 1, 4}, 8: {5, 4, 2}}
    for c in range(3):
        for p in range(27):
            nz = set(np.nonzero(star[c, p])[0].tolist())
            allowed = vel_cols[p] if p in vel_cols else {6, 7, 8}
            assert nz <= allowed, (c, p, nz)
        assert np.count_nonzero(star[c]) == 51  # the count nz_counts_visco uses


def test_visco_source_pattern_matches_the_kernel():
    """E: normal stresses <- the 9 normal memory variables, shear stresses <- 3 (their own
    component in each mechanism), memory variables <- themselves, velocities: none."""
    E = physics.source_matrix(np.array([0.6, 6.0, 60.0]), np.array([1.0, 2.0, 3.0]), np.array([0.5, 0.7, 0.9]))
    assert np.count_nonzero(E) == 54
    for p in range(27):
        nz = set(np.nonzero(E[p])[0].tolist())
        if p < 3:
            assert nz == {9 + 6 * l + t for l in range(3) for t in range(3)}, p
        elif p < 6:
            assert nz == {9 + 6 * l + p for l in range(3)}, p
        elif p < 9:
            assert nz == set(), p
        else:
            assert nz == {p}, p


def test_visco_nz_counts_formula():
    """nz_counts_visco at N = 1 recomputed from the oracle's matrix counts."""
    from math import comb
    from paper_1903_11521_b200.gen import tables
    N = 1
    t = tables.load(N)
    B, Bt = t["B"], t["Bt"]
    nK = sum(int(np.count_nonzero(np.array(k))) for k in t["K"])
    nR = sum(int(np.count_nonzero(np.array(r))) for r in t["R"])
    nf = sum(int(np.count_nonzero(np.array(f))) for f in t["f"]) / 3.0
    star, _ = _visco_star()
    ns = np.count_nonzero(star[0])
    ne = 54
    loc = (N * (27 * nK + 3 * ns * B + ne * B) + 27 * B * (N + 1)
           + 27 * nK + 3 * ns * comb(N + 2, 3) + ne * B + 9 * nR + 4 * Bt * 27 * 9 + 27 * nR)
    neigh = 9 * 4 * nf + 4 * Bt * 27 * 9 + 27 * nR
    got = kernels.nz_counts_visco(N)
    assert got["local_flops"] == 2 * loc + 27 * B
    assert got["flops"] == 2 * (loc + neigh) + 2 * 27 * B
