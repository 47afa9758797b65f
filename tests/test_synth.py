"""The seeded input generators (synth/): determinism, ranges, counter-addressability."""
import numpy as np

import synth


def test_uniform_is_counter_based_and_in_range():
    a = synth.uniform(0, synth.STREAM_DOFS, np.arange(1000, dtype=np.uint64), -1.0, 1.0)
    b = synth.uniform(0, synth.STREAM_DOFS, np.arange(500, 1000, dtype=np.uint64), -1.0, 1.0)
    assert np.array_equal(a[500:], b)
    assert a.min() >= -1.0 and a.max() < 1.0
    c = synth.uniform(1, synth.STREAM_DOFS, np.arange(1000, dtype=np.uint64), -1.0, 1.0)
    assert not np.array_equal(a, c)
    assert abs(a.mean()) < 0.1


def test_dofs_subrange_matches_full():
    cfg = synth.CONFIGS["c0"]
    full = synth.dofs(cfg)
    part = synth.dofs(cfg, first=100, count=7)
    assert full.shape == (384, 9, 10)
    assert np.array_equal(full[100:107], part)


def test_kuhn_mesh_layout():
    xyz, vid = synth.kuhn_mesh(4, 4, 4)
    assert xyz.shape == (384, 4, 3) and vid.shape == (384, 4)
    J = np.stack([xyz[:, 1] - xyz[:, 0], xyz[:, 2] - xyz[:, 0], xyz[:, 3] - xyz[:, 0]], 2)
    assert (np.linalg.det(J) > 0).all()
    # z-major element order: the first 6*16 elements are the cubes of layer z = 0
    assert (xyz[: 6 * 16, :, 2].mean(1) < 1.2).all()
    assert vid.max() == 63


def test_material_distributions():
    cfg = synth.CONFIGS["c0"]
    m = synth.material(cfg)
    assert (m[:, 0] >= 2000).all() and (m[:, 0] <= 3000).all()
    assert (m[:, 1] >= 3000).all() and (m[:, 1] <= 6000).all()
    assert np.allclose(m[:, 2], m[:, 1] / np.sqrt(3))
    two = synth.CONFIGS["c2"].replica(4)
    m2 = synth.material(two)
    upper = np.arange(two.n_elements) // (6 * 16) >= 2
    assert (m2[upper, 1] <= 2500).all() and (m2[~upper, 1] >= 4000).all()
