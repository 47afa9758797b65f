"""Element geometry, face matching and the neighbour relation.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The paper's scheme references the neighbour relation through Neigh(sigma, mu),
Face(sigma, mu) and Rot(sigma, mu) without fixing conventions (reading R7):

* local faces are the outward-oriented vertex triples FACES = (0,2,1), (0,1,3), (0,3,2), (1,2,3);
* two element faces are the same face iff their sorted topological vertex-id triples match
  (every face must match exactly twice; the meshes are periodic);
* Neigh = nb, Face = j (the neighbour's local face), Rot = h = position of the element's
  face-first-vertex id inside the neighbour's face-j triple.

The oracle's own neighbour flux does not use (j, h): it maps each face point to the
neighbour through the vertex-id correspondence (``neighbour_vertex_map``).  (nb, j, h) are
produced here only for the bit-exact table check against the library.

Geometry (reading R5/R7): J = [x1-x0 | x2-x0 | x3-x0], det J > 0 required; face area |S_i|
and outward unit normal n_i from the cross product of the face edges in triple order.
"""
from __future__ import annotations

import numpy as np

from .matrices import FACES


def geometry(elem_xyz):
    """(J (E,3,3), Jinv (E,3,3), detJ (E,), area (E,4), normal (E,4,3))."""
    x = np.asarray(elem_xyz, dtype=np.float64)
    J = np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]], axis=2)
    detJ = np.linalg.det(J)
    if np.any(detJ <= 0):
        raise ValueError("element with det J <= 0")
    Jinv = np.linalg.inv(J)
    area = np.zeros((x.shape[0], 4))
    normal = np.zeros((x.shape[0], 4, 3))
    for i, (a, b, c) in enumerate(FACES):
        cr = np.cross(x[:, b] - x[:, a], x[:, c] - x[:, a])
        nrm = np.linalg.norm(cr, axis=1)
        area[:, i] = 0.5 * nrm
        normal[:, i] = cr / nrm[:, None]
    return J, Jinv, detJ, area, normal


def match_faces(elem_vid):
    """nb (E,4) int64 by sorted vertex-id triples; raises if a face is not matched exactly twice."""
    vid = np.asarray(elem_vid)
    E = vid.shape[0]
    table = {}
    for e in range(E):
        for i, tri in enumerate(FACES):
            key = tuple(sorted(int(vid[e, t]) for t in tri))
            table.setdefault(key, []).append((e, i))
    nb = np.full((E, 4), -1, dtype=np.int64)
    for key, lst in table.items():
        if len(lst) != 2:
            raise ValueError(f"face {key} matched {len(lst)} times")
        (e1, i1), (e2, i2) = lst
        if e1 == e2:
            raise ValueError("element is its own neighbour")
        nb[e1, i1] = e2
        nb[e2, i2] = e1
    return nb


def neighbour_vertex_map(elem_vid, e, i, n):
    """Local vertex indices in element n of the vertices (a, b, c) of face i of element e."""
    ids = [int(elem_vid[e, t]) for t in FACES[i]]
    nv = [int(v) for v in elem_vid[n]]
    return tuple(nv.index(v) for v in ids)


def neighbour_table(elem_vid):
    """(nb, j, h), each (E,4): Neigh, Face, Rot of P:1342 under reading R7 (brute force)."""
    vid = np.asarray(elem_vid)
    nb = match_faces(vid)
    E = vid.shape[0]
    j = np.zeros((E, 4), dtype=np.int8)
    h = np.zeros((E, 4), dtype=np.int8)
    for e in range(E):
        for i in range(4):
            n = nb[e, i]
            mine = [int(vid[e, t]) for t in FACES[i]]
            found = None
            for jj, tri in enumerate(FACES):
                theirs = [int(vid[n, t]) for t in tri]
                if sorted(theirs) == sorted(mine):
                    found = jj
                    break
            theirs = [int(vid[n, t]) for t in FACES[found]]
            j[e, i] = found
            h[e, i] = theirs.index(mine[0])
    return nb, j, h
