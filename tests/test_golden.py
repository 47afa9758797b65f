"""The oracle against the values the paper prints (tests/golden/paper_values.txt, each record
with its PAPER.md citation).  CPU only; nothing here touches the CUDA path."""
import os
from math import comb

import numpy as np
import pytest

import synth
from oracle import basis, matrices, step

HERE = os.path.dirname(os.path.abspath(__file__))


def _records():
    out = []
    for line in open(os.path.join(HERE, "golden", "paper_values.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, args, value, cite = [f.strip() for f in line.split("|", 3)]
        assert cite.startswith("P:"), f"record without a citation: {line}"
        out.append((key, args, value))
    return out


RECORDS = _records()
ORDERS = [1, 2, 3, 4, 5]


def _formula(expr, **names):
    return eval(expr, {"C": comb, "__builtins__": {}}, names)  # the fixture's own closed forms


def test_fixture_has_every_record_kind():
    assert {k for k, _, _ in RECORDS} == {
        "basis_functions", "face_basis_functions", "derivative_nonzeros", "khat_nonzero_columns",
        "volume_flop_saving", "ktilde_pattern", "quantities_elastic"}


@pytest.mark.parametrize("N", ORDERS)
def test_basis_sizes(N):
    (b,) = [v for k, _, v in RECORDS if k == "basis_functions"]
    (bt,) = [v for k, _, v in RECORDS if k == "face_basis_functions"]
    assert basis.n_basis(N) == _formula(b, N=N) == len(basis.tet_index(N))
    assert basis.n_face_basis(N) == _formula(bt, N=N) == len(basis.tri_index(N))
    for i in range(4):
        assert matrices.lift_matrix(N, i).shape == (_formula(b, N=N), _formula(bt, N=N))


@pytest.mark.parametrize("N", ORDERS)
def test_khat_columns_and_ktilde_pattern(N):
    (cols,) = [v for k, _, v in RECORDS if k == "khat_nonzero_columns"]
    nz = _formula(cols, N=N)
    Kh, Kt = matrices.volume_matrices(N), matrices.derivative_matrices(N)
    used = np.zeros(Kh.shape[2], bool)
    for c in range(3):
        used |= (Kh[c] != 0).any(axis=0)
        assert ((Kt[c] != 0) == (Kh[c].T != 0)).all()  # ktilde_pattern record
    assert used[:nz].all() and not used[nz:].any()
    for key, args, value in RECORDS:  # the printed savings: 50 % (fourth order), 37.5 % (sixth)
        if key == "volume_flop_saving" and int(args) == N:
            assert 1.0 - nz / basis.n_basis(N) == pytest.approx(float(value), abs=1e-15)


@pytest.mark.parametrize("N", [2, 3, 5])
def test_derivative_nonzero_counts_on_random_data(N):
    """The CK recursion of the oracle on seeded random DOFs: D^delta has exactly the printed
    number of rows that can be nonzero, and (generic data) every one of them is."""
    (expr,) = [v for k, _, v in RECORDS if k == "derivative_nonzeros"]
    (P,) = [int(v) for k, _, v in RECORDS if k == "quantities_elastic"]
    small = synth.CONFIGS["c0"].replica(3, name="c0-r3")  # 3^3 cubes: the smallest periodic mesh
    cfg = small.__class__(**{**small.__dict__, "N": N})
    xyz, vid = synth.kuhn_mesh(cfg.nx, cfg.ny, cfg.nz, seed=cfg.seed)
    prob = step.setup(N, xyz, vid, synth.material(cfg))
    Q = step.to_internal(synth.dofs(cfg))
    assert Q.shape[1:] == (basis.n_basis(N), P)
    _, Ds = step.time_integral(prob, Q, cfg.dt)
    assert len(Ds) == N + 1
    for delta, D in enumerate(Ds):
        rows = _formula(expr, N=N, delta=delta)
        assert not D[:, rows:, :].any()
        assert (np.abs(D[:, :rows, :]).max(axis=(0, 2)) > 0).all()
