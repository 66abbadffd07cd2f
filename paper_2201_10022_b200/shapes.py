"""Procedural closed meshes for scenes, tests and the benchmark configs.

`box_mesh` and `icosphere_mesh` follow the reference generators
(`shapes.py:32-99`) vertex-for-vertex so seeded scenes match the oracle;
`torus_mesh` is new (the chainmail config needs it).
"""
from __future__ import annotations

import numpy as np

from .mesh import SurfaceMesh

__all__ = ["box_mesh", "icosphere_mesh", "torus_mesh", "hexahedron_mesh", "prism_mesh", "wedge_mesh"]

# corners of [-1, 1]^3 and the 12 CCW-outward triangles (two per face)
_CORNERS = np.array([[x, y, z] for z in (-1, 1) for (x, y) in ((-1, -1), (1, -1), (1, 1), (-1, 1))],
                    dtype=float)
_FACES = np.array([
    [0, 2, 1], [0, 3, 2], [4, 5, 6], [4, 6, 7],
    [0, 1, 5], [0, 5, 4], [2, 3, 7], [2, 7, 6],
    [0, 4, 7], [0, 7, 3], [1, 2, 6], [1, 6, 5],
], dtype=np.int64)


def box_mesh(size=1.0, center=(0.0, 0.0, 0.0)) -> SurfaceMesh:
    half = 0.5 * np.broadcast_to(np.asarray(size, dtype=float), (3,))
    return SurfaceMesh(_CORNERS * half + np.asarray(center, dtype=float), _FACES)


def hexahedron_mesh(corners) -> SurfaceMesh:
    return SurfaceMesh(np.asarray(corners, dtype=float).reshape(8, 3), _FACES)


def icosphere_mesh(radius=1.0, subdivisions=1, center=(0.0, 0.0, 0.0)) -> SurfaceMesh:
    """Unit icosahedron refined `subdivisions` times (20*4^k triangles)."""
    g = (1.0 + np.sqrt(5.0)) / 2.0
    base = np.array([
        (-1, g, 0), (1, g, 0), (-1, -g, 0), (1, -g, 0),
        (0, -1, g), (0, 1, g), (0, -1, -g), (0, 1, -g),
        (g, 0, -1), (g, 0, 1), (-g, 0, -1), (-g, 0, 1),
    ], dtype=float)
    base /= np.linalg.norm(base[0])
    faces = [
        (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
        (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
        (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
        (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
    ]
    pts = list(base)
    for _ in range(subdivisions):
        mid: dict[tuple[int, int], int] = {}

        def split(i, j):
            k = (i, j) if i < j else (j, i)
            if k not in mid:
                m = pts[i] + pts[j]
                pts.append(m / np.linalg.norm(m))
                mid[k] = len(pts) - 1
            return mid[k]

        nxt = []
        for a, b, c in faces:
            ab, bc, ca = split(a, b), split(b, c), split(c, a)
            nxt.extend([(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)])
        faces = nxt
    v = np.asarray(pts) * radius + np.asarray(center, dtype=float)
    return SurfaceMesh(v, np.asarray(faces, dtype=np.int64))


def torus_mesh(major=0.1, minor=0.02, n_major=24, n_minor=8, center=(0.0, 0.0, 0.0)) -> SurfaceMesh:
    """Closed torus in the xy plane: n_major*n_minor vertices, 2x that many triangles."""
    u = 2.0 * np.pi * np.arange(n_major) / n_major
    v = 2.0 * np.pi * np.arange(n_minor) / n_minor
    U, Vv = np.meshgrid(u, v, indexing="ij")
    rr = major + minor * np.cos(Vv)
    pts = np.stack([rr * np.cos(U), rr * np.sin(U), minor * np.sin(Vv)], axis=-1).reshape(-1, 3)
    idx = np.arange(n_major * n_minor).reshape(n_major, n_minor)
    i0 = idx
    i1 = np.roll(idx, -1, axis=0)
    j1 = np.roll(idx, -1, axis=1)
    k1 = np.roll(np.roll(idx, -1, axis=0), -1, axis=1)
    tris = np.concatenate([
        np.stack([i0, i1, k1], axis=-1).reshape(-1, 3),
        np.stack([i0, k1, j1], axis=-1).reshape(-1, 3),
    ])
    m = SurfaceMesh(pts + np.asarray(center, dtype=float), tris)
    a, b, c = (m.vertices[m.triangles[:, k]] for k in range(3))
    if np.einsum("ij,ij->i", a - pts.mean(0) * 0, np.cross(b, c)).sum() < 0:
        m = SurfaceMesh(m.vertices, m.triangles[:, ::-1])
    return m


def _outward(m: SurfaceMesh) -> SurfaceMesh:
    """Flip every triangle when the signed volume is negative."""
    a, b, c = (m.vertices[m.triangles[:, k]] for k in range(3))
    if np.einsum("ij,ij->i", a, np.cross(b, c)).sum() < 0:
        return SurfaceMesh(m.vertices, m.triangles[:, ::-1])
    return m


def prism_mesh(n_sides=6, radius=1.0, height=1.0, axis=2) -> SurfaceMesh:
    """Closed regular prism about a coordinate axis (reference shapes.py:125-152 layout:
    bottom ring, top ring, bottom centre, top centre)."""
    n = int(n_sides)
    t = 2.0 * np.pi * np.arange(n) / n
    plane = [k for k in range(3) if k != axis]
    v = np.zeros((2 * n + 2, 3))
    for ring, h in ((0, -0.5 * height), (1, 0.5 * height)):
        v[ring * n:(ring + 1) * n, plane[0]] = radius * np.cos(t)
        v[ring * n:(ring + 1) * n, plane[1]] = radius * np.sin(t)
        v[ring * n:(ring + 1) * n, axis] = h
    v[2 * n, axis], v[2 * n + 1, axis] = -0.5 * height, 0.5 * height
    tris = []
    for i in range(n):
        j = (i + 1) % n
        tris += [(i, j, n + j), (i, n + j, n + i), (2 * n, j, i), (2 * n + 1, n + i, n + j)]
    return _outward(SurfaceMesh(v, np.asarray(tris, dtype=np.int64)))


def wedge_mesh(theta0, theta1, r_inner, r_outer, depth) -> SurfaceMesh:
    """Annular-sector prism in the xz plane extruded along y, centred on its corner mean
    (reference shapes.py:96-122; corners in the box corner order)."""
    def at(th, r, y):
        return [r * np.cos(th), y, r * np.sin(th)]

    c = []
    for y in (-0.5 * depth, 0.5 * depth):
        c += [at(theta0, r_inner, y), at(theta1, r_inner, y), at(theta1, r_outer, y), at(theta0, r_outer, y)]
    c = np.asarray(c, dtype=float)
    return _outward(hexahedron_mesh(c - c.mean(axis=0)))
