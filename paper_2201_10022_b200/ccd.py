"""Additive CCD along linear trajectories (drop-in for `stiffbody.ccd`, ccd.py:1-153).

`accd_toi_batch` and `step_filter` run kernel K5 (csrc/abd_misc.cuh
accd_query): same iteration as the reference, numpy arithmetic order, the
global step bound as an ordered atomic min with the exact early-exit rule
(a query stops once its t exceeds the current minimum).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = ["CcdQuery", "accd_toi", "accd_toi_batch", "step_filter", "DEFAULT_SLACK", "MAX_ITERATIONS"]

DEFAULT_SLACK = 0.1
MAX_ITERATIONS = 512
ADVANCE_EPS = 1e-12


@dataclass(frozen=True)
class CcdQuery:
    kind: str
    x: np.ndarray
    dx: np.ndarray
    slack: float = DEFAULT_SLACK
    t_max: float = 1.0

    def __post_init__(self):
        object.__setattr__(self, "x", np.asarray(self.x, dtype=float).reshape(4, 3))
        object.__setattr__(self, "dx", np.asarray(self.dx, dtype=float).reshape(4, 3))
        if self.kind not in ("vertex-face", "edge-edge"):
            raise ValueError(f"unknown CCD query kind {self.kind!r}")
        if not (0.0 < self.slack < 1.0):
            raise ValueError("slack must be in (0, 1)")
        if not (0.0 < self.t_max <= 1.0):
            raise ValueError("t_max must be in (0, 1]")


def accd_toi_batch(kind, x, dx, slack=DEFAULT_SLACK, t_max=1.0, max_iterations=MAX_ITERATIONS):
    x = np.asarray(x, dtype=float).reshape(-1, 4, 3)
    if len(x) == 0:
        return np.zeros(0)
    return _native.accd_batch(kind, x, dx, slack, t_max, max_iterations)


def accd_toi(query: CcdQuery) -> float:
    return float(accd_toi_batch(query.kind, query.x[None], query.dx[None], query.slack, query.t_max)[0])


def step_filter(bodies, q_all, delta_q, candidates, slack=DEFAULT_SLACK) -> float:
    """Largest certified step fraction over all candidates (ccd.py:130-153)."""
    if len(candidates) == 0:
        return 1.0
    sc = _native.scene_for(bodies)
    sc.set_candidates(candidates)
    out = C.c_double(1.0)
    _native.check(_native.lib().abd_step_filter(sc.ptr, sc.q(q_all), sc.q(delta_q), float(slack), C.byref(out)))
    return float(out.value)
