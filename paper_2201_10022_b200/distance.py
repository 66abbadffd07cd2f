"""Squared-distance kernels (drop-in for `stiffbody.distance`, distance.py:1-401).

All batch entry points run the sm_100a kernels in csrc/abd_math.cuh and
csrc/abd_pair.cuh through the C-ABI; closest-point classification and d^2
reproduce numpy's operation order bit-for-bit.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _native

__all__ = [
    "PTRegion", "EERegion", "DistanceResult", "point_triangle_distance_sq", "edge_edge_distance_sq",
    "point_triangle_closest", "edge_edge_closest", "pair_distance_gradients", "ee_mollifier",
    "ee_mollifier_grad_hess", "DEFAULT_MOLLIFIER_SCALE",
]

DEFAULT_MOLLIFIER_SCALE = 1e-3


class PTRegion(IntEnum):
    VERT0 = 0
    VERT1 = 1
    VERT2 = 2
    EDGE01 = 3
    EDGE12 = 4
    EDGE20 = 5
    INTERIOR = 6


class EERegion(IntEnum):
    """3 * (edge-a feature) + (edge-b feature); 0/1 endpoint, 2 interior."""

    A0_B0 = 0
    A0_B1 = 1
    A0_INT = 2
    A1_B0 = 3
    A1_B1 = 4
    A1_INT = 5
    INT_B0 = 6
    INT_B1 = 7
    INT_INT = 8


@dataclass(frozen=True)
class DistanceResult:
    d_sq: float
    region: IntEnum
    ee_parallel_mollifier: float = 1.0


def _stack(*pts):
    arrs = np.broadcast_arrays(*(np.atleast_2d(np.asarray(p, dtype=float)) for p in pts))
    return np.stack(arrs, axis=1)


def point_triangle_closest(p, t0, t1, t2):
    """(d_sq, region, bary) for batched point-triangle pairs (distance.py:86-150)."""
    return _native.pt_closest(_stack(p, t0, t1, t2))


def edge_edge_closest(a0, a1, b0, b1):
    """(d_sq, region, s, t) for batched segment pairs (distance.py:167-204)."""
    return _native.ee_closest(_stack(a0, a1, b0, b1))


def point_triangle_distance_sq(p, t0, t1, t2) -> DistanceResult:
    a, b, c = (np.asarray(v, dtype=float) for v in (t0, t1, t2))
    if np.linalg.norm(np.cross(b - a, c - a)) == 0.0:
        raise ValueError("degenerate triangle in point_triangle_distance_sq")
    d2, reg, _ = point_triangle_closest(p, a, b, c)
    return DistanceResult(float(d2[0]), PTRegion(int(reg[0])))


def ee_mollifier(a0, a1, b0, b1, eps_x=None):
    z = _stack(a0, a1, b0, b1)
    if eps_x is None:
        u = z[:, 1] - z[:, 0]
        v = z[:, 3] - z[:, 2]
        eps_x = DEFAULT_MOLLIFIER_SCALE * np.einsum("ij,ij->i", u, u) * np.einsum("ij,ij->i", v, v)
    return _native.mollifier(z, eps_x, derivs=False)


def edge_edge_distance_sq(a0, a1, b0, b1, eps_x=None) -> DistanceResult:
    pts = [np.asarray(v, dtype=float) for v in (a0, a1, b0, b1)]
    if np.linalg.norm(pts[1] - pts[0]) == 0.0 or np.linalg.norm(pts[3] - pts[2]) == 0.0:
        raise ValueError("zero-length edge in edge_edge_distance_sq")
    d2, reg, _, _ = edge_edge_closest(*pts)
    mol = ee_mollifier(*pts, eps_x)
    return DistanceResult(float(d2[0]), EERegion(int(reg[0])), float(mol[0]))


def pair_distance_gradients(kind: str, z: np.ndarray):
    """(d2, grad (N,12), hess (N,12,12), region, gamma) (distance.py:291-339)."""
    if kind not in ("vf", "ee"):
        raise ValueError(f"unknown pair kind {kind!r}")
    return _native.d2_derivatives(kind, z)


def ee_mollifier_grad_hess(z: np.ndarray, eps_x: np.ndarray):
    """(value, grad (N,12), hess (N,12,12)) (distance.py:342-401)."""
    return _native.mollifier(z, eps_x, derivs=True)
