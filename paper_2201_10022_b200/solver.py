"""Implicit-Euler projected-Newton stepping (drop-in for `stiffbody.solver`).

`advance_step` runs the whole Newton step on the device through one C-ABI
call (`abd_advance_step`, csrc/driver.cu): q, q_dot, candidates, friction,
the BSR system and the PCG workspace stay resident in HBM; only scalars
cross per iteration.  The finer-grained entries (`assemble`, `ip_value`,
`line_search`, `solve_newton_system`, `compute_q_tilde`) run the same
kernels individually.  Reference: /root/reference/pkg/src/stiffbody/solver.py.
"""
from __future__ import annotations

import ctypes as C
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .body import BodyMaterial, GeneralizedMass
from .contact import CandidateSet, CollisionBody, FrictionData
from .sparse import BlockSparseMatrix

__all__ = [
    "StepParams", "SystemModel", "SimState", "StepStats", "StepFailure", "IncrementalPotentialState",
    "compute_q_tilde", "ip_value", "assemble", "solve_newton_system", "line_search", "advance_step",
    "global_min_distance",
]

PCG_MAX_ITERS = 50000


class StepFailure(RuntimeError):
    """Line-search underflow (solver.py:69-74)."""

    def __init__(self, message, diagnostics=None):
        super().__init__(message)
        self.diagnostics = diagnostics or {}


@dataclass
class StepParams:
    dt: float
    d_hat: float = 1e-3
    kappa_barrier: float = 1e4
    mu: float = 0.0
    epsilon_v: float = 1e-3
    newton_tol: float = 1e-2
    max_newton_iters: int = 64
    friction_outer_iters: int = 1
    ccd_slack: float = 0.1
    ccd_step_scale: float = 0.9
    workers: int = 1  # accepted for API compatibility; the GPU path has no host pool
    audit_iterates: bool = False
    # Newton linear solve: "cholesky" = device sparse block Cholesky + refinement (the
    # reference's BlockCholesky.solve_refined), "pcg" = block-Jacobi PCG to 1e-8 residual
    linear_solver: str = "cholesky"

    def __post_init__(self):
        if self.dt <= 0 or self.d_hat <= 0 or self.newton_tol <= 0:
            raise ValueError("dt, d_hat and newton_tol must be positive")
        if self.mu < 0:
            raise ValueError("friction coefficient must be >= 0")
        if self.linear_solver not in ("cholesky", "pcg"):
            raise ValueError("linear_solver must be 'cholesky' or 'pcg'")


@dataclass
class SystemModel:
    bodies: list
    gmass: list
    materials: list
    force_fn: object = None
    reduction: object = None

    def __post_init__(self):
        self.dynamic = np.array([b.dynamic for b in self.bodies], dtype=bool)
        self.dyn_indices = np.nonzero(self.dynamic)[0]
        self.n_dyn = len(self.dyn_indices)
        self.slot_of = {int(b): s for s, b in enumerate(self.dyn_indices)}
        for b in self.dyn_indices:
            if self.gmass[b] is None or self.materials[b] is None:
                raise ValueError(f"dynamic body {b} missing mass or material")
        self._scene = None

    def forces(self, step_index, t_next, q_all) -> np.ndarray:
        if self.force_fn is None:
            return np.zeros((len(self.bodies), 12))
        return np.asarray(self.force_fn(step_index, t_next, q_all), dtype=float)

    def gpu_scene(self) -> "_native.Scene":
        """Device context with geometry, masses and stiffness (created on first use)."""
        if self._scene is None:
            masses = [g.matrix if g is not None else None for g in self.gmass]
            stiff = [m.stiffness_scale if m is not None else None for m in self.materials]
            self._scene = _native.Scene(self.bodies, masses, stiff)
        return self._scene


@dataclass
class SimState:
    q: np.ndarray
    q_dot: np.ndarray
    time: float = 0.0
    step_index: int = 0
    u: np.ndarray | None = None
    u_dot: np.ndarray | None = None

    def copy(self) -> "SimState":
        return SimState(self.q.copy(), self.q_dot.copy(), self.time, self.step_index,
                        None if self.u is None else self.u.copy(),
                        None if self.u_dot is None else self.u_dot.copy())


@dataclass
class IncrementalPotentialState:
    q_prev: np.ndarray
    q_dot_prev: np.ndarray
    q_tilde: np.ndarray
    friction: FrictionData
    candidates: CandidateSet
    model: SystemModel


@dataclass
class StepStats:
    step: int
    iterations: int
    converged: bool
    min_distance: float
    candidates: int
    ip_value: float
    max_ortho_error: float
    energy_trace: list = field(default_factory=list)
    min_iterate_distance: float = np.inf
    timings: dict = field(default_factory=dict)
    pcg_iterations: int = 0


def _sync_ip(sc, ip: IncrementalPotentialState):
    sc.set_candidates(ip.candidates)
    sc.set_friction(ip.friction)


def compute_q_tilde(model: SystemModel, state: SimState, params: StepParams, forces: np.ndarray) -> np.ndarray:
    """q + dt q_dot + dt^2 M^-1 f per dynamic body (solver.py:179-190)."""
    sc = model.gpu_scene()
    out = np.empty((len(model.bodies), 12))
    _native.check(_native.lib().abd_compute_q_tilde(sc.ptr, sc.q(state.q), sc.q(state.q_dot), sc.q(forces),
                                                    float(params.dt), out))
    return out


def ip_value(q_all, ip: IncrementalPotentialState, params: StepParams) -> float:
    """Incremental potential (solver.py:193-205), kernels K1 + K6."""
    sc = ip.model.gpu_scene()
    _sync_ip(sc, ip)
    out = C.c_double(0.0)
    _native.check(_native.lib().abd_ip_value(sc.ptr, sc.q(q_all), sc.q(ip.q_tilde), float(params.dt),
                                             float(params.kappa_barrier), float(params.d_hat),
                                             float(params.epsilon_v), C.byref(out)))
    return float(out.value)


def assemble(q_all, ip: IncrementalPotentialState, params: StepParams, timings: dict | None = None):
    """Gradient and block-sparse Hessian (solver.py:257-342), kernels K1 + K3 + K7."""
    model = ip.model
    sc = model.gpu_scene()
    _sync_ip(sc, ip)
    tic = time.perf_counter()
    n_off = C.c_int64(0)
    _native.check(_native.lib().abd_assemble(sc.ptr, sc.q(q_all), sc.q(ip.q_tilde), float(params.dt),
                                             float(params.kappa_barrier), float(params.d_hat),
                                             float(params.epsilon_v), C.byref(n_off)))
    if timings is not None:
        timings["narrow_phase"] = timings.get("narrow_phase", 0.0) + time.perf_counter() - tic
    n = model.n_dyn
    grad = np.empty(12 * n)
    diag = np.empty((n, 12, 12))
    keys = np.empty((n_off.value, 2), dtype=np.int64)
    off = np.empty((n_off.value, 12, 12))
    _native.check(_native.lib().abd_get_system(sc.ptr, grad, diag, keys, off))
    H = BlockSparseMatrix(n, [tuple(k) for k in keys])
    H.diag[:] = diag
    for k, blk in zip(keys, off):
        H.off[(int(k[0]), int(k[1]))][:] = blk
    return grad, H


def solve_newton_system(hessian: BlockSparseMatrix, gradient: np.ndarray) -> np.ndarray:
    """H dq = -g by the device sparse block Cholesky with iterative refinement to 1e-8 relative
    residual (solver.py:345-348; sparse.py:90-161)."""
    return hessian.factor().solve_refined(-np.asarray(gradient, dtype=float), rel_tol=1e-8)


def line_search(q_all, delta_q, ip: IncrementalPotentialState, params: StepParams, e0: float | None = None,
                timings: dict | None = None):
    """CCD-capped backtracking (solver.py:358-393), kernels K5 + K6."""
    from .ccd import step_filter

    model = ip.model
    tic = time.perf_counter()
    alpha_max = step_filter(model.bodies, q_all, delta_q, ip.candidates, slack=params.ccd_slack)
    if timings is not None:
        timings["ccd"] = timings.get("ccd", 0.0) + time.perf_counter() - tic
    alpha = 1.0 if alpha_max >= 1.0 else min(1.0, params.ccd_step_scale * alpha_max)
    if e0 is None:
        e0 = ip_value(q_all, ip, params)
    while True:
        e = ip_value(q_all + alpha * delta_q, ip, params)
        if e < e0:
            return alpha, e
        alpha *= 0.5
        if alpha < 1e-12:
            raise StepFailure("line search underflow (no descent below alpha = 1e-12)",
                              diagnostics={"e0": e0, "candidates": len(ip.candidates), "alpha_max": alpha_max})


def global_min_distance(bodies, q_all, skip_static_pairs=True) -> float:
    """Exact minimum inter-body distance (solver.py:396-473), on the GPU."""
    sc = _native.scene_for(bodies)
    out = C.c_double(0.0)
    _native.check(_native.lib().abd_global_min_distance(sc.ptr, sc.q(q_all), int(bool(skip_static_pairs)),
                                                        C.byref(out)))
    return float(out.value)


def step_params_c(params: StepParams, min_distance=True, pcg_rel_tol=1e-8,
                  pcg_max_iters=PCG_MAX_ITERS) -> "_native.StepParamsC":
    return _native.StepParamsC(
        dt=params.dt, d_hat=params.d_hat, kappa_barrier=params.kappa_barrier, mu=params.mu,
        epsilon_v=params.epsilon_v, newton_tol=params.newton_tol, ccd_slack=params.ccd_slack,
        ccd_step_scale=params.ccd_step_scale, pcg_rel_tol=pcg_rel_tol,
        max_newton_iters=params.max_newton_iters, friction_outer_iters=params.friction_outer_iters,
        pcg_max_iters=pcg_max_iters, compute_min_distance=1 if min_distance else 0,
        linear_solver=1 if params.linear_solver == "pcg" else 0, audit_iterates=1 if params.audit_iterates else 0)


def _sync_reduction(model: SystemModel, sc) -> None:
    """Device copy of the joint reduction's T (abd_set_reduction), refreshed when the model's
    reduction object or its T changes; removed when the model has none."""
    red = model.reduction
    key = None if red is None else (id(red), id(red.T), red.T.shape)
    if getattr(sc, "_red_key", None) == key:
        return
    if red is None:
        _native.check(_native.lib().abd_set_reduction(sc.ptr, 0, None))
    else:
        T = np.ascontiguousarray(red.T, dtype=np.float64)
        if T.shape[0] != 12 * model.n_dyn:
            raise ValueError(f"reduction T has {T.shape[0]} rows, expected 12 x {model.n_dyn} dynamic bodies")
        _native.check(_native.lib().abd_set_reduction(sc.ptr, T.shape[1], T.ctypes.data))
        sc._red_T = T  # keep the host copy alive with the key
    sc._red_key = key


def advance_step(model: SystemModel, state: SimState, params: StepParams):
    """One implicit-Euler step (solver.py:493-628) fully on the device; with a joint reduction
    the Newton direction comes from T^T H T on the device (solver.py:479-490)."""
    sc = model.gpu_scene()
    _sync_reduction(model, sc)
    B = len(model.bodies)
    q0 = np.ascontiguousarray(state.q, dtype=np.float64).reshape(B, 12)
    qd = np.ascontiguousarray(state.q_dot, dtype=np.float64).reshape(B, 12)
    t_next = state.time + params.dt
    forces = np.ascontiguousarray(model.forces(state.step_index, t_next, q0), dtype=np.float64).reshape(B, 12)
    L = _native.lib()
    _native.check(L.abd_set_state(sc.ptr, q0.ctypes.data, qd.ctypes.data))
    cp = step_params_c(params)
    st = _native.StepStatsC()
    trace = np.zeros(max(1, params.max_newton_iters * max(1, params.friction_outer_iters)))
    rc = L.abd_advance_step(sc.ptr, forces.ctypes.data, C.byref(cp), C.byref(st), trace.ctypes.data)
    if rc == _native.ABD_ERR_STEP_FAILURE:
        raise StepFailure(L.abd_last_error().decode(), diagnostics={"step": state.step_index})
    _native.check(rc)
    q = np.empty((B, 12))
    qdn = np.empty((B, 12))
    _native.check(L.abd_get_state(sc.ptr, q.ctypes.data, qdn.ctypes.data))
    for _ in range(st.nondescent_fallbacks):
        warnings.warn("projected system produced a non-descent direction; falling back to steepest descent",
                      RuntimeWarning)
    if not st.converged:
        warnings.warn(f"step {state.step_index}: Newton did not converge in {params.max_newton_iters} "
                      f"iterations (|dq|/dt = {st.last_dq_over_dt:.3e})", RuntimeWarning)
    # (not state.copy(): q and q_dot are replaced, copying them first costs ~0.7 ms on the 10k pile)
    new_state = SimState(q, qdn, state.time, state.step_index,
                         None if state.u is None else state.u.copy(),
                         None if state.u_dot is None else state.u_dot.copy())
    if model.reduction is not None:  # solver.py:595-600 (host bookkeeping of the reduced state)
        new_state.u = model.reduction.extract_u(q[model.dyn_indices].reshape(-1))
        new_state.u_dot = model.reduction.extract_u_rate(qdn[model.dyn_indices].reshape(-1))
    new_state.time = t_next
    new_state.step_index = state.step_index + 1
    timings = {"broad_phase": st.t_broad * 1e-3, "narrow_phase": 0.0, "assembly": st.t_assemble * 1e-3,
               "solve": st.t_solve * 1e-3, "ccd": st.t_ccd * 1e-3, "line_search": st.t_line_search * 1e-3,
               "total": st.t_total * 1e-3}
    stats = StepStats(
        step=state.step_index, iterations=st.iterations, converged=bool(st.converged),
        min_distance=st.min_distance, candidates=int(st.candidates), ip_value=st.ip_value,
        max_ortho_error=st.max_ortho_error, energy_trace=list(trace[:st.iterations]),
        min_iterate_distance=st.min_iterate_distance,
        timings=timings, pcg_iterations=st.pcg_iters_total)
    return new_state, stats
