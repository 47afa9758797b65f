"""Pins of the LTS oracle (oracle/lts.py, reading R26; NEXT-2): reduction to global time
stepping when all elements share a cluster, interval additivity of the Taylor integral,
steady constant state and plane-wave convergence at order N+1 with mixed clusters."""
from math import comb

import numpy as np
import pytest

import synth
from oracle import lts, step
from tests.test_oracle_step import _problem, _project

SMALL = synth.CONFIGS["c0"].replica(3, name="c0-r3")


def test_single_cluster_is_global_time_stepping():
    prob, *_ = _problem(SMALL)
    Q = step.to_internal(synth.dofs(SMALL))
    dt = SMALL.dt / 4
    fine = lts.lts_cycle(prob, Q, dt, np.zeros(SMALL.n_elements, int))
    gts2 = step.step(prob, step.step(prob, Q, dt), dt)
    assert np.abs(fine - gts2).max() <= 1e-13 * np.abs(gts2).max()
    coarse = lts.lts_cycle(prob, Q, dt, np.ones(SMALL.n_elements, int))
    gts1 = step.step(prob, Q, 2 * dt)
    assert np.abs(coarse - gts1).max() <= 1e-13 * np.abs(gts1).max()


def test_interval_integral_additivity():
    prob, *_ = _problem(SMALL)
    Q = step.to_internal(synth.dofs(SMALL))
    dt = 1e-4
    I, Ds = step.time_integral(prob, Q, dt)
    assert np.abs(lts.interval_integral(Ds, 0.0, dt) - I).max() <= 1e-14 * np.abs(I).max()
    a = lts.interval_integral(Ds, 0.0, 0.3 * dt) + lts.interval_integral(Ds, 0.3 * dt, dt)
    assert np.abs(a - I).max() <= 1e-14 * np.abs(I).max()


def test_constant_state_is_steady_with_mixed_clusters():
    prob, *_ = _problem(SMALL, homogeneous=True)
    rng = np.random.default_rng(0)
    Q = np.zeros((SMALL.n_elements, comb(SMALL.N + 3, 3), 9))
    Q[:, 0, :] = rng.uniform(-1, 1, 9)
    cl = rng.integers(0, 2, SMALL.n_elements)
    out = lts.lts_cycle(prob, Q, SMALL.dt / 4, cl)
    assert np.abs(out - Q).max() < 1e-8  # volume terms of ~1e6 cancel (as for GTS)


def test_linearity():
    prob, *_ = _problem(SMALL)
    rng = np.random.default_rng(1)
    Q1 = step.to_internal(synth.dofs(SMALL))
    Q2 = rng.uniform(-1, 1, Q1.shape)
    cl = rng.integers(0, 2, SMALL.n_elements)
    dt = SMALL.dt / 4
    lhs = lts.lts_cycle(prob, 0.5 * Q1 - 3 * Q2, dt, cl)
    rhs = 0.5 * lts.lts_cycle(prob, Q1, dt, cl) - 3 * lts.lts_cycle(prob, Q2, dt, cl)
    assert np.abs(lhs - rhs).max() < 1e-13 * np.abs(lhs).max()


def _plane_wave_lts_error(N, n):
    rho, vp = 2500.0, 5000.0
    vs = vp / np.sqrt(3.0)
    from oracle import physics
    lam, mu = physics.lame(rho, vp, vs)
    A = physics.jacobians(rho, lam, mu)
    k = 2 * np.pi / n * np.array([1.0, 1.0, 0.0])
    w, X = np.linalg.eig(np.einsum("d,dpq->pq", k, A))
    idx = np.argmax(w.real)
    omega, r = w[idx].real, X[:, idx].real
    r = r / np.abs(r).max()

    def exact(x, t):
        return np.sin(x @ k - omega * t)[:, None] * r[None, :]

    xyz, vid = synth.kuhn_mesh(n, n, n, seed=3)
    E = xyz.shape[0]
    prob = step.setup(N, xyz, vid, np.tile([rho, vp, vs], (E, 1)))
    Q, (pts, wq, phi, x) = _project(N, xyz, lambda y: exact(y, 0.0))
    # clusters: the lower half of the domain (z < n/2) is fine, the upper half coarse
    cl = (xyz[:, :, 2].mean(1) >= n / 2).astype(int)
    T = 0.2 * 2 * np.pi / omega
    cycles = 2 * n
    Q = lts.lts(prob, Q, T / (2 * cycles), cl, cycles)
    qh = np.einsum("rk,ekp->erp", phi, Q)
    qe = exact(x.reshape(-1, 3), T).reshape(qh.shape)
    from oracle import mesh
    detJ = mesh.geometry(xyz)[2]
    scale = np.r_[np.full(6, np.abs(r[:6]).max()), np.full(3, np.abs(r[6:]).max())][None, None, :]
    err = np.sqrt((detJ[:, None, None] * wq[None, :, None] * ((qh - qe) / scale) ** 2).sum())
    ref = np.sqrt((detJ[:, None, None] * wq[None, :, None] * (qe / scale) ** 2).sum())
    return err / ref


@pytest.mark.parametrize("N", [1, 2])
def test_plane_wave_convergence_with_lts(N):
    """A plane wave crossing the fine/coarse cluster interface converges at order N+1 (the
    same check as the paper's validation of the scheme)."""
    e4, e8 = _plane_wave_lts_error(N, 4), _plane_wave_lts_error(N, 8)
    rate = np.log2(e4 / e8)
    assert rate > N + 1 - 0.3, (e4, e8, rate)
