"""Barrier contact, broad phase and lagged friction (drop-in for `stiffbody.contact`).

Every compute entry runs on the GPU (kernels K2, K3, K6, K7 in csrc/):
candidate sets, energies and per-pair blocks are produced by the sm_100a
kernels and copied back into the reference's host record types.
Reference: /root/reference/pkg/src/stiffbody/contact.py.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .mesh import SurfaceMesh

__all__ = [
    "CollisionBody", "ContactPair", "CandidateSet", "PairBlocks", "FrictionData", "BarrierDomainError",
    "barrier", "barrier_d1", "barrier_d2", "barrier_distance_form", "broad_phase", "contact_energy",
    "contact_gradient_hessian", "candidate_min_distance_sq", "friction_precompute", "friction_energy",
    "friction_gradient_hessian", "world_positions_all",
]


class BarrierDomainError(ValueError):
    """Barrier evaluated at non-positive squared distance (contact.py:53-58)."""


def _barrier(d_sq, d_hat, k):
    s = np.asarray(d_sq, dtype=float)
    out = _native.barrier_batch(s.reshape(-1), d_hat)[k]
    return out.reshape(s.shape)


def barrier(d_sq, d_hat):
    """B(d) = -(d - d_hat)^2 ln(d / d_hat) for d < d_hat, else 0; argument s = d^2."""
    return _barrier(d_sq, d_hat, 0)


def barrier_d1(d_sq, d_hat):
    return _barrier(d_sq, d_hat, 1)


def barrier_d2(d_sq, d_hat):
    return _barrier(d_sq, d_hat, 2)


def barrier_distance_form(d, d_hat):
    """Plain-distance oracle form of the barrier (contact.py:79-84; host helper)."""
    d = np.asarray(d, dtype=float)
    with np.errstate(divide="ignore", invalid="ignore"):
        v = -((d - d_hat) ** 2) * np.log(d / d_hat)
    return np.where(d < d_hat, v, 0.0)


@dataclass(frozen=True)
class CollisionBody:
    rest: np.ndarray
    triangles: np.ndarray
    edges: np.ndarray
    edge_rest_len_sq: np.ndarray
    dynamic: bool = True

    @classmethod
    def from_mesh(cls, mesh: SurfaceMesh, dynamic: bool = True) -> "CollisionBody":
        return cls(mesh.vertices, mesh.triangles, mesh.edges, mesh.edge_rest_length_sq(), dynamic)


def world_positions_all(bodies, q_all) -> list:
    """Per-body world vertices rest @ A^T + p (contact.py:149-153) on the GPU
    (abd_world_vertices, the reference's rounding)."""
    sc = _native.scene_for(bodies)
    X = np.empty((sum(len(b.rest) for b in bodies), 3))
    _native.check(_native.lib().abd_world_vertices(sc.ptr, sc.q(q_all), X))
    off = np.cumsum([0] + [len(b.rest) for b in bodies])
    return [X[off[k]:off[k + 1]] for k in range(len(bodies))]


@dataclass(frozen=True)
class ContactPair:
    kind: str
    body_a: int
    body_b: int
    prim_a: int
    prim_b: int

    def __post_init__(self):
        if self.body_a == self.body_b:
            raise ValueError("contact pairs are inter-body only")


@dataclass
class CandidateSet:
    vf: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), dtype=np.int64))
    ee: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), dtype=np.int64))
    overlap_pairs: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), dtype=np.int64))
    box_tests: int = 0

    def __len__(self) -> int:
        return len(self.vf) + len(self.ee)

    def pairs(self) -> list:
        out = [ContactPair("vertex-face", int(r[0]), int(r[2]), int(r[1]), int(r[3])) for r in self.vf]
        out += [ContactPair("edge-edge", int(r[0]), int(r[2]), int(r[1]), int(r[3])) for r in self.ee]
        return out


@dataclass
class PairBlocks:
    body_a: np.ndarray
    body_b: np.ndarray
    grad: np.ndarray
    hess: np.ndarray
    d_sq: np.ndarray

    @classmethod
    def empty(cls) -> "PairBlocks":
        z = np.zeros(0, dtype=np.int64)
        return cls(z, z, np.zeros((0, 24)), np.zeros((0, 24, 24)), np.zeros(0))


@dataclass
class FrictionData:
    body_a: np.ndarray
    body_b: np.ndarray
    lam: np.ndarray
    mu: float
    tangent_map: np.ndarray
    offset: np.ndarray
    basis: np.ndarray

    def __len__(self) -> int:
        return len(self.lam)

    @classmethod
    def empty(cls, mu=0.0) -> "FrictionData":
        z = np.zeros(0, dtype=np.int64)
        return cls(z, z, np.zeros(0), mu, np.zeros((0, 2, 24)), np.zeros((0, 2)), np.zeros((0, 3, 2)))


# ---------------------------------------------------------------------------

def broad_phase(bodies, q_start, q_end, d_hat) -> CandidateSet:
    """Exact candidate set of the reference broad phase (contact.py:338-412), GPU kernel K2."""
    sc = _native.scene_for(bodies)
    vf, ee, ov = sc.broad_phase(q_start, q_end, d_hat)
    cs = CandidateSet(vf, ee, ov, 0)
    sc.adopt_candidates(cs)
    return cs


def contact_energy(bodies, q_all, candidates: CandidateSet, kappa, d_hat) -> float:
    sc = _native.scene_for(bodies)
    sc.set_candidates(candidates)
    out = C.c_double(0.0)
    _native.check(_native.lib().abd_contact_energy(sc.ptr, sc.q(q_all), float(kappa), float(d_hat), C.byref(out)))
    return float(out.value)


def candidate_min_distance_sq(bodies, q_all, candidates: CandidateSet):
    if len(candidates) == 0:
        return None
    sc = _native.scene_for(bodies)
    sc.set_candidates(candidates)
    out = C.c_double(0.0)
    _native.check(_native.lib().abd_candidate_min_d2(sc.ptr, sc.q(q_all), C.byref(out)))
    return float(out.value)


def _fetch_blocks(sc, n) -> PairBlocks:
    a = np.empty(n, dtype=np.int64)
    b = np.empty(n, dtype=np.int64)
    g = np.empty((n, 24))
    h = np.empty((n, 24, 24))
    d2 = np.empty(n)
    _native.check(_native.lib().abd_get_pair_blocks(sc.ptr, a, b, g, h, d2))
    return PairBlocks(a, b, g, h, d2)


def contact_gradient_hessian(bodies, q_all, candidates: CandidateSet, kappa, d_hat,
                             project: bool = True) -> PairBlocks:
    """Per active pair g24 and (projected) H24 (contact.py:646-675), GPU kernel K3."""
    sc = _native.scene_for(bodies)
    sc.set_candidates(candidates)
    n = C.c_int64(0)
    _native.check(_native.lib().abd_contact_gradient_hessian(sc.ptr, sc.q(q_all), float(kappa), float(d_hat),
                                                             int(bool(project)), C.byref(n)))
    return _fetch_blocks(sc, n.value)


def friction_precompute(bodies, q_prev, candidates: CandidateSet, kappa, d_hat, mu) -> FrictionData:
    """Lagged friction terms at q_prev (contact.py:722-790), GPU kernel K7."""
    if mu < 0:
        raise ValueError("friction coefficient must be >= 0")
    sc = _native.scene_for(bodies)
    sc.set_candidates(candidates)
    n = C.c_int64(0)
    _native.check(_native.lib().abd_friction_precompute(sc.ptr, sc.q(q_prev), float(kappa), float(d_hat),
                                                        float(mu), C.byref(n)))
    m = n.value
    a, b = np.empty(m, dtype=np.int64), np.empty(m, dtype=np.int64)
    lam, tm, off, basis = np.empty(m), np.empty((m, 2, 24)), np.empty((m, 2)), np.empty((m, 3, 2))
    _native.check(_native.lib().abd_get_friction(sc.ptr, a, b, lam, tm, off, basis))
    return FrictionData(a, b, lam, float(mu), tm, off, basis)


def friction_energy(q_all, data: FrictionData, dt, epsilon_v) -> float:
    if len(data) == 0:
        return 0.0
    q = np.asarray(q_all, dtype=float).reshape(-1, 12)
    e, _, _ = _native.friction_batch(data, q, np.ones(len(q), dtype=bool), dt, epsilon_v, False, False)
    return e


def friction_gradient_hessian(q_all, data: FrictionData, dt, epsilon_v, dynamic,
                              project: bool = True) -> PairBlocks:
    if len(data) == 0:
        return PairBlocks.empty()
    _, g, h = _native.friction_batch(data, q_all, dynamic, dt, epsilon_v, project, True)
    return PairBlocks(data.body_a.copy(), data.body_b.copy(), g, h, np.full(len(data), np.inf))
