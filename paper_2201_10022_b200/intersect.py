"""Exact intersection audit on the GPU (drop-in for stiffbody.intersect and the
scene audit's pair test; intersect.py:18-52, scene.py:627-698).

`triangles_intersect_batch` runs the closed-triangle separating-axis test in
`abd_tri_intersect_batch`; `intersecting_body_pairs` checks every box-overlapping
body pair of a state (triangle SAT, then ray-parity containment) in
`abd_intersecting_pairs` (csrc/k_audit.cu).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native

__all__ = ["triangles_intersect", "triangles_intersect_batch", "intersecting_body_pairs"]


def triangles_intersect_batch(tri_a: np.ndarray, tri_b: np.ndarray) -> np.ndarray:
    """(N,3,3) x (N,3,3) -> bool (N,): closed triangles intersect (touching counts)."""
    a = _native.f64(tri_a).reshape(-1, 3, 3)
    b = _native.f64(tri_b).reshape(-1, 3, 3)
    if a.shape != b.shape:
        raise ValueError("tri_a and tri_b must have the same shape")
    out = np.zeros(len(a), dtype=np.uint8)
    if len(a):
        _native.check(_native.lib().abd_tri_intersect_batch(len(a), a, b, out))
    return out.astype(bool)


def triangles_intersect(tri_a, tri_b) -> bool:
    a = np.asarray(tri_a, dtype=float).reshape(3, 3)
    b = np.asarray(tri_b, dtype=float).reshape(3, 3)
    for t in (a, b):
        if np.linalg.norm(np.cross(t[1] - t[0], t[2] - t[0])) == 0.0:
            raise ValueError("degenerate triangle in triangles_intersect")
    return bool(triangles_intersect_batch(a[None], b[None])[0])


def intersecting_body_pairs(bodies, q_all, skip_pair=None) -> list:
    """Body pairs (i, j), i < j, whose closed surfaces intersect or where one body
    contains the other, at generalized coordinates q_all (scene.py:652-698)."""
    sc = _native.scene_for(bodies)
    q = sc.q(q_all)
    n = C.c_int64(0)
    cap = 4096
    while True:
        pairs = np.zeros((cap, 2), dtype=np.int64)
        _native.check(_native.lib().abd_intersecting_pairs(sc.ptr, q, cap, pairs, C.byref(n)))
        if n.value <= cap:
            break
        cap = n.value
    res = [(int(i), int(j)) for i, j in pairs[:n.value]]
    if skip_pair is not None:
        res = [(i, j) for i, j in res if not skip_pair(i, j)]
    return res
