"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This module holds NONE of the method's arithmetic: it only draws numbers and builds the
synthetic Kuhn meshes that stand in for the paper's workloads (the SeisSol performance
reproducer with "random initial data" and the LOH.1 mesh, are
not available).  Recipe:

* Mesh: nx x ny x nz unit cubes (h = 1), each split into 6 Kuhn tetrahedra, periodic in
  all three axes.  Vertex ids are periodic lattice ids vid = x + nx (y + ny z).  Each
  periodic vertex is jittered by U[-0.1, 0.1] h per axis; an element's coordinates are its
  unwrapped lattice positions plus the jitter of each vertex id.  Tet t of a cube is the
  axis permutation pi_t (itertools order): v0 = corner, v1 = v0 + e_pi0, v2 = v1 + e_pi1,
  v3 = corner + (1,1,1); for odd pi, v1 and v2 are swapped so det J > 0.  Element order
  e = 6 (x + nx (y + ny z)) + t  (z-major: contiguous z-slabs).
* Material per element: rho ~ U[2000, 3000], vp ~ U[3000, 6000], vs = vp / sqrt(3)
  (config "two_layer": cubes with z >= nz/2 draw vp ~ U[1500, 2500], the others
  vp ~ U[4000, 6000]).
* DOFs Q ~ U[-1, 1] for every (element, quantity, basis function).
* Viscoelastic: omega_l = 2 pi f_l, f = (0.1, 1, 10) Hz; Ylam_l = lam / 150, Ymu_l = mu / 150
  (these two are *inputs*, computed here from the drawn material).
* dt = 0.2 h / vp_hi with vp_hi the upper bound of the vp distribution.

Random numbers: counter-based SplitMix64.  For (seed, stream, index):
  base = mix64(seed * 2^8 + stream),  x = mix64(base + (index + 1) * 0x9E3779B97F4A7C15),
  U[a, b] = a + (b - a) * (x >> 11) * 2^-53.
So any single value can be regenerated on its own (sampled parity at full size).
"""
from __future__ import annotations

import itertools
import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

STREAM_JITTER = 1
STREAM_MATERIAL = 2
STREAM_DOFS = 3
STREAM_VPERM = 4

KUHN_PERMS = tuple(itertools.permutations(range(3)))
# the 12 even permutations of an element's 4 local vertices (keep det J > 0)
EVEN_PERMS4 = tuple(p for p in itertools.permutations(range(4))
                    if sum(1 for i in range(4) for j in range(i + 1, 4) if p[i] > p[j]) % 2 == 0)


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _base(seed, stream):
    return _mix64(np.uint64((int(seed) << 8) + int(stream)))


def uniform(seed, stream, index, a, b):
    """U[a,b] draws for integer counter array ``index`` (vectorised)."""
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = _mix64(_base(seed, stream) + (idx + np.uint64(1)) * GOLDEN)
    u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return a + (b - a) * u


def uniform_range(seed, stream, start, count, a, b, out=None, threads=None):
    """U[a,b] draws for counters start .. start+count-1 into a flat float64 array."""
    if out is None:
        out = np.empty(count, dtype=np.float64)
    chunk = 1 << 22
    nthreads = threads or min(32, os.cpu_count() or 1)

    def work(off):
        n = min(chunk, count - off)
        out[off:off + n] = uniform(seed, stream, np.arange(start + off, start + off + n, dtype=np.uint64), a, b)

    offs = range(0, count, chunk)
    if count > chunk and nthreads > 1:
        with ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(work, offs))
    else:
        for o in offs:
            work(o)
    return out


@dataclass(frozen=True)
class Config:
    name: str
    N: int            # polynomial degree
    P: int            # quantities (9 elastic, 27 viscoelastic)
    precision: int    # 8 = fp64, 4 = fp32
    nx: int
    ny: int
    nz: int
    steps: int
    material: str = "uniform"  # or "two_layer"
    seed: int = 0
    jitter: float = 0.1
    vperm: bool = False  # per-element random even vertex permutation (all 48 (i, j, h) cases)

    @property
    def n_elements(self):
        return 6 * self.nx * self.ny * self.nz

    @property
    def B(self):
        return math.comb(self.N + 3, 3)

    @property
    def vp_hi(self):
        return 6000.0

    @property
    def dt(self):
        return 0.2 * 1.0 / self.vp_hi

    def replica(self, nx, ny=None, nz=None, name=None, steps=None):
        """Same N / P / precision / distributions on a smaller periodic mesh."""
        return Config(name or f"{self.name}-r{nx}", self.N, self.P, self.precision, nx,
                      ny or nx, nz or nx, steps if steps is not None else self.steps,
                      self.material, self.seed, self.jitter, self.vperm)

    def with_(self, **kw):
        return Config(**{**self.__dict__, **kw})


# BASELINE.json configs[0..4]
CONFIGS = {
    "c0": Config("c0", 2, 9, 8, 4, 4, 4, 1),
    "c1": Config("c1", 5, 9, 8, 64, 64, 64, 10),
    "c2": Config("c2", 6, 9, 4, 96, 96, 64, 10, material="two_layer"),
    "c3": Config("c3", 4, 27, 8, 64, 64, 48, 10),
    "c4": Config("c4", 5, 9, 8, 128, 128, 128, 20),
}


def kuhn_mesh(nx, ny, nz, seed=0, jitter=0.1, vperm=False):
    """(elem_xyz (E,4,3) float64, elem_vid (E,4) int64) of the periodic jittered Kuhn mesh.

    vperm: reorder each element's 4 vertices by a seeded random even permutation (det J
    keeps its sign).  The Kuhn order alone produces only 6 of the 48 (face i, neighbour
    face j, orientation h) cases of the neighbour relation; with vperm every case
    occurs on meshes of a few hundred elements, as on the paper's reproducer with random
    neighbour relations."""
    nv = nx * ny * nz
    jit = uniform_range(seed, STREAM_JITTER, 0, 3 * nv, -jitter, jitter).reshape(nv, 3)
    # cube corners in element order
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    corner = np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1)  # cube index c = x + nx(y + ny z)
    nc = corner.shape[0]
    offs = np.zeros((6, 4, 3), dtype=np.int64)
    for t, pi in enumerate(KUHN_PERMS):
        e0 = np.zeros(3, dtype=np.int64)
        e1 = e0.copy()
        e1[pi[0]] = 1
        e2 = e1.copy()
        e2[pi[1]] = 1
        e3 = np.ones(3, dtype=np.int64)
        v = [e0, e1, e2, e3]
        # parity of the permutation
        inv = sum(1 for i in range(3) for j in range(i + 1, 3) if pi[i] > pi[j])
        if inv % 2 == 1:
            v[1], v[2] = v[2], v[1]
        offs[t] = np.stack(v)
    pos = corner[:, None, None, :] + offs[None, :, :, :]  # (nc, 6, 4, 3) unwrapped lattice positions
    pos = pos.reshape(nc * 6, 4, 3)
    w = pos % np.array([nx, ny, nz])
    vid = w[..., 0] + nx * (w[..., 1] + ny * w[..., 2])
    xyz = pos.astype(np.float64) + jit[vid]
    vid = vid.astype(np.int64)
    if vperm:
        E = xyz.shape[0]
        u = uniform(seed, STREAM_VPERM, np.arange(E, dtype=np.uint64), 0.0, 12.0)
        perm = np.asarray(EVEN_PERMS4, dtype=np.int64)[np.minimum(u.astype(np.int64), 11)]
        xyz = np.take_along_axis(xyz, perm[:, :, None], axis=1)
        vid = np.take_along_axis(vid, perm, axis=1)
    return xyz, vid


def mesh(cfg: "Config"):
    """kuhn_mesh of a config (its seed, jitter and vertex-permutation flag)."""
    return kuhn_mesh(cfg.nx, cfg.ny, cfg.nz, seed=cfg.seed, jitter=cfg.jitter, vperm=cfg.vperm)


def material(cfg: Config, first=0, count=None):
    """(count, 3) array of (rho, vp, vs) for elements first..first+count-1."""
    E = cfg.n_elements if count is None else count
    e = np.arange(first, first + E, dtype=np.uint64)
    rho = uniform(cfg.seed, STREAM_MATERIAL, e * np.uint64(4) + np.uint64(0), 2000.0, 3000.0)
    if cfg.material == "two_layer":
        cz = (e // np.uint64(6 * cfg.nx * cfg.ny)).astype(np.int64)
        upper = cz >= cfg.nz // 2
        u = uniform(cfg.seed, STREAM_MATERIAL, e * np.uint64(4) + np.uint64(1), 0.0, 1.0)
        vp = np.where(upper, 1500.0 + 1000.0 * u, 4000.0 + 2000.0 * u)
    else:
        vp = uniform(cfg.seed, STREAM_MATERIAL, e * np.uint64(4) + np.uint64(1), 3000.0, 6000.0)
    vs = vp / math.sqrt(3.0)
    return np.stack([rho, vp, vs], axis=1)


MECH_FREQ_HZ = (0.1, 1.0, 10.0)
Y_FACTOR = 1.0 / 150.0


def anelastic(cfg: Config, mat):
    """(omega (3,), Y (E,3,2)) inputs of the viscoelastic configs (reading R15)."""
    omega = np.array([2.0 * math.pi * f for f in MECH_FREQ_HZ])
    rho, vp, vs = mat[:, 0], mat[:, 1], mat[:, 2]
    mu = rho * vs * vs
    lam = rho * vp * vp - 2.0 * mu
    Y = np.zeros((mat.shape[0], 3, 2))
    Y[:, :, 0] = (lam * Y_FACTOR)[:, None]
    Y[:, :, 1] = (mu * Y_FACTOR)[:, None]
    return omega, Y


def dofs(cfg: Config, first=0, count=None, out=None, threads=None):
    """Q in the canonical layout (count, P, B), U[-1,1], float64."""
    E = cfg.n_elements if count is None else count
    n = E * cfg.P * cfg.B
    flat = uniform_range(cfg.seed, STREAM_DOFS, first * cfg.P * cfg.B, n, -1.0, 1.0,
                         out=None if out is None else out.reshape(-1), threads=threads)
    return flat.reshape(E, cfg.P, cfg.B)


# ---- LinA (NEXT-3): ADER-DG-SEM acoustics on a uniform periodic grid of cuboids
STREAM_LINA_MAT = 5
STREAM_LINA_DOFS = 6


@dataclass(frozen=True)
class LinaConfig:
    name: str
    N: int            # polynomial degree per axis (order N+1 <= 8)
    nx: int
    ny: int
    nz: int
    steps: int
    h: tuple = (1.0, 1.0, 1.0)
    seed: int = 0

    @property
    def n_elements(self):
        return self.nx * self.ny * self.nz

    @property
    def c_max(self):
        return math.sqrt(1e10 / 1000.0)

    @property
    def dt(self):
        # well inside the ADER-DG-SEM stability bound ~ h / (c (2N+1) d)
        return 0.2 * min(self.h) / (self.c_max * (2 * self.N + 1) * 3)

    def with_(self, **kw):
        return LinaConfig(**{**self.__dict__, **kw})


# LinA's paper runs orders 8-32 in 2D/3D; here 3D order 8 on 64^3 elements
LINA_CONFIGS = {
    "lina": LinaConfig("lina", 7, 64, 64, 64, 10),
    "lina-small": LinaConfig("lina-small", 3, 4, 3, 5, 2),
}


def lina_material(cfg: LinaConfig):
    """(E, 2) = (rho ~ U[1000, 3000], K ~ U[1e9, 1e10]) per element."""
    e = np.arange(cfg.n_elements, dtype=np.uint64)
    rho = uniform(cfg.seed, STREAM_LINA_MAT, 2 * e, 1000.0, 3000.0)
    K = uniform(cfg.seed, STREAM_LINA_MAT, 2 * e + np.uint64(1), 1e9, 1e10)
    return np.stack([rho, K], axis=1)


def lina_dofs(cfg: LinaConfig, first=0, count=None):
    """Q in the ABI layout (count, 4, n, n, n): p ~ U[-1e6, 1e6] (Pa), velocities U[-1, 1]."""
    E = cfg.n_elements if count is None else count
    n = cfg.N + 1
    flat = uniform_range(cfg.seed, STREAM_LINA_DOFS, first * 4 * n ** 3, E * 4 * n ** 3, -1.0, 1.0)
    Q = flat.reshape(E, 4, n, n, n)
    Q[:, 0] *= 1e6
    return Q
