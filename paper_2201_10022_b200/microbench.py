"""BASELINE config 2: the kernel microbenchmark through the scene path.

100k bodies, 10M VF + 10M EE synthetic pairs (`scenes.microbench_pairs`), every
pair active (d ~ U(0, d_hat)).  One "run" = `assemble` (K1 body terms, K3 pair
grad/Hessian + J^T H J + PSD projection, the deterministic BSR reduction; the
reference's `assemble`, solver.py:257-342) followed by the block-Jacobi PCG on
the resulting SPD 12x12-block BSR to 1e-8 relative residual
(`solve_newton_system` contract, solver.py:345-348 / sparse.py:149-161).

The synthetic pairs carry their own 4 rest points, so each pair's primitives
become a small triangle-soup piece of its bodies' rest meshes: the VF vertex is
a vertex of body_a, the face a triangle of body_b, each EE edge an edge of its
body.  The resulting arrays are exactly the `abd_scene_create` layout, so the
benchmark runs the production kernels (no benchmark-only kernels), with the
candidate set uploaded through `abd_set_candidates` and the BSR pattern = the
Morton +-1..4 body graph given as overlap pairs (solver.py:270-281).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .body import GeneralizedMass

__all__ = ["soup_arrays", "PairSystem", "unit_cube_mass"]


def unit_cube_mass(density=1000.0):
    """Generalised mass of a centred unit cube (mass = rho, second moment rho/12 I)."""
    return GeneralizedMass.from_moments(density, np.zeros(3), np.eye(3) * density / 12.0).matrix


def _layout(owner, n_bodies):
    """Stable per-body order of records: (offsets (B+1), new global index per record)."""
    order = np.argsort(owner, kind="stable")
    inv = np.empty(len(owner), dtype=np.int64)
    inv[order] = np.arange(len(owner), dtype=np.int64)
    off = np.zeros(n_bodies + 1, dtype=np.int64)
    np.cumsum(np.bincount(owner, minlength=n_bodies), out=off[1:])
    return order, inv, off


def morton_pattern(order):
    """Body pairs (i < j) of the Morton +-1..4 neighbour graph (8 neighbours per row)."""
    B = len(order)
    ps = []
    for k in range(1, 5):
        a, b = order[:B - k], order[k:]
        ps.append(np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1))
    ov = np.concatenate(ps).astype(np.int64)
    ov = np.unique(ov, axis=0)
    return ov


def soup_arrays(data):
    """Scene + candidate arrays for `scenes.microbench_pairs` output.

    Returns dict(v_off, e_off, t_off, rest, edges, tris, el2, vf, ee, ov, vf_perm, ee_perm)
    (rows grouped by body pair; row k is generated pair perm[k]): local
    vertex indices in edges/tris, candidate rows (body, prim, body, prim) in the
    reference's CandidateSet convention (contact.py:175-204; EE with body_a < body_b).
    """
    q = data["q"]
    B = len(q)
    vf, ee = data["vf"], data["ee"]
    nv, ne = len(vf["body_a"]), len(ee["body_a"])
    va = vf["body_a"].astype(np.int64)
    vb = vf["body_b"].astype(np.int64)
    ea = ee["body_a"].astype(np.int64)
    eb = ee["body_b"].astype(np.int64)
    er = ee["rest"]
    swap = ea > eb
    if swap.any():
        ea, eb = np.where(swap, eb, ea), np.where(swap, ea, eb)
        er = er.copy()
        er[swap] = er[swap][:, [2, 3, 0, 1]]
    # vertex records: VF vertex | VF triangle corners | EE edge-a ends | EE edge-b ends
    owner = np.concatenate([va, np.repeat(vb, 3), np.repeat(ea, 2), np.repeat(eb, 2)])
    rest_rec = np.concatenate([vf["rest"][:, 0], vf["rest"][:, 1:].reshape(-1, 3),
                               er[:, :2].reshape(-1, 3), er[:, 2:].reshape(-1, 3)])
    vorder, vinv, v_off = _layout(owner, B)
    rest = rest_rec[vorder]
    local = vinv - v_off[owner]
    del rest_rec, vorder, vinv
    o1 = nv
    o2 = o1 + 3 * nv
    o3 = o2 + 2 * ne
    v_local = local[:nv]
    tri_local = local[o1:o2].reshape(nv, 3)
    ea_local = local[o2:o3].reshape(ne, 2)
    eb_local = local[o3:].reshape(ne, 2)
    # triangles (one per VF pair, owned by body_b)
    torder, tinv, t_off = _layout(vb, B)
    tris = tri_local[torder]
    t_idx = tinv - t_off[vb]
    # edges (two per EE pair)
    eowner = np.concatenate([ea, eb])
    eorder, einv, e_off = _layout(eowner, B)
    e_rec = np.concatenate([ea_local, eb_local])
    edges = e_rec[eorder]
    e_idx = einv - e_off[eowner]
    # rest lengths (mesh.py edge_rest_len_sq: squared length of the rest edge)
    gl = edges + np.repeat(v_off[:-1], np.diff(e_off))[:, None]
    dv = rest[gl[:, 1]] - rest[gl[:, 0]]
    el2 = dv[:, 0] * dv[:, 0] + dv[:, 1] * dv[:, 1] + dv[:, 2] * dv[:, 2]
    vf_rows = np.stack([va, v_local, vb, t_idx], axis=1)
    ee_rows = np.stack([ea, e_idx[:ne], eb, e_idx[ne:]], axis=1)
    # candidates grouped by body pair, as the broad phase emits them (overlap-pair
    # order): consecutive pairs of one body pair form the runs the fused assembly sums
    vf_perm = np.lexsort((np.arange(len(vf_rows)), vf_rows[:, 2], vf_rows[:, 0]))
    ee_perm = np.lexsort((np.arange(len(ee_rows)), ee_rows[:, 2], ee_rows[:, 0]))
    vf_rows, ee_rows = vf_rows[vf_perm], ee_rows[ee_perm]
    ov = morton_pattern(data["order"])
    return dict(v_off=v_off, e_off=e_off, t_off=t_off, rest=rest, edges=edges, tris=tris, el2=el2,
                vf=vf_rows, ee=ee_rows, ov=ov, vf_perm=vf_perm, ee_perm=ee_perm)


class PairSystem:
    """Device context for config 2: soup scene + resident candidates + q, q_tilde."""

    def __init__(self, data, density=1000.0, kappa_ortho=1e8, dt=0.01, gravity=(0.0, 0.0, -9.8),
                 kappa_barrier=1e4):
        arrs = soup_arrays(data)
        q = np.ascontiguousarray(data["q"], dtype=np.float64)
        B = len(q)
        self.B = B
        self.dt = dt
        self.kappa = kappa_barrier
        self.d_hat = float(data["d_hat"])
        M1 = unit_cube_mass(density)
        mass = np.broadcast_to(M1, (B, 12, 12))
        stiff = np.full(B, kappa_ortho * 1.0)
        self.scene = _native.Scene.from_arrays(arrs["v_off"], arrs["e_off"], arrs["t_off"], arrs["rest"],
                                               arrs["edges"], arrs["tris"], arrs["el2"], np.ones(B, np.uint8),
                                               np.ascontiguousarray(mass), stiff)
        self.n_vf, self.n_ee, self.n_ov = len(arrs["vf"]), len(arrs["ee"]), len(arrs["ov"])
        self.arrays = arrs
        L = _native.lib()
        _native.check(L.abd_set_candidates(self.scene.ptr, self.n_vf, _native.i64a(arrs["vf"]), self.n_ee,
                                           _native.i64a(arrs["ee"]), self.n_ov, _native.i64a(arrs["ov"])))
        self.q = q
        g = np.asarray(gravity, dtype=float)
        f = np.zeros((B, 12))
        f[:, :3] = M1[0, 0] * g  # centred body: zero first moment, so the affine rows vanish
        self.forces = f
        self.q_tilde = np.empty((B, 12))
        _native.check(L.abd_compute_q_tilde(self.scene.ptr, q, np.zeros((B, 12)), f, float(dt), self.q_tilde))

    def assemble(self):
        """K1 + K3 + reduction into the resident gradient + BSR; returns n_off."""
        n_off = C.c_int64(0)
        _native.check(_native.lib().abd_assemble(self.scene.ptr, self.q, self.q_tilde, float(self.dt),
                                                 float(self.kappa), float(self.d_hat), 1e-3, C.byref(n_off)))
        self.n_off = n_off.value
        return self.n_off

    def solve(self, rel_tol=1e-8, max_iters=100000):
        """Block-Jacobi PCG on the resident system: (dx, iterations, relative residual)."""
        dx = np.empty(12 * self.B)
        it, rel = C.c_int(0), C.c_double(0.0)
        _native.check(_native.lib().abd_solve_resident(self.scene.ptr, float(rel_tol), int(max_iters), dx,
                                                       C.byref(it), C.byref(rel)))
        return dx, it.value, rel.value

    def system(self):
        """(grad, diag (n,12,12), keys (n_off,2), off (n_off,12,12)) copied to the host."""
        n_off = getattr(self, "n_off", None)
        if n_off is None:
            raise RuntimeError("call assemble() first")
        grad = np.empty(12 * self.B)
        diag = np.empty((self.B, 12, 12))
        keys = np.empty((n_off, 2), dtype=np.int64)
        off = np.empty((n_off, 12, 12))
        _native.check(_native.lib().abd_get_system(self.scene.ptr, grad, diag, keys, off))
        return grad, diag, keys, off
