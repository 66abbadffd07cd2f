"""Seeded generators for the BASELINE.json configurations (physical units, z up).

Each generator returns a `SceneSpec` of plain arrays (rest meshes, dynamic
flags, q0, q_dot0, materials, step parameters).  Scenes are built directly
in metres as `SystemModel`s (no unit-box normalisation).
Resolved ambiguities are stated inline and in DESIGN.md.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import SurfaceMesh
from .shapes import box_mesh, icosphere_mesh, torus_mesh

__all__ = ["SceneSpec", "box_stack", "cube_drop", "icosphere_pile", "chainmail",
           "random_rotation", "rot_z", "microbench_pairs"]


@dataclass
class SceneSpec:
    name: str
    meshes: list
    dynamic: np.ndarray
    q0: np.ndarray
    q_dot0: np.ndarray
    density: float
    kappa_ortho: float
    params: dict
    steps: int
    gravity: tuple = (0.0, 0.0, -9.8)
    meta: dict = field(default_factory=dict)

    def build(self):
        """(SystemModel, SimState, StepParams) of the product package."""
        from .body import BodyMaterial, external_generalized_force, mass_matrix
        from .contact import CollisionBody
        from .solver import SimState, StepParams, SystemModel

        bodies, gms, mats = [], [], []
        cache = {}
        for mesh, dyn in zip(self.meshes, self.dynamic):
            bodies.append(CollisionBody.from_mesh(mesh, dynamic=bool(dyn)))
            if not dyn:
                gms.append(None)
                mats.append(None)
                continue
            key = id(mesh)
            if key not in cache:
                cache[key] = mass_matrix(mesh, self.density)
            gm, vol = cache[key]
            gms.append(gm)
            mats.append(BodyMaterial(self.density, self.kappa_ortho, vol))
        model = SystemModel(bodies, gms, mats)
        g = np.asarray(self.gravity, dtype=float)
        fixed = np.zeros((len(bodies), 12))
        for b in model.dyn_indices:
            fixed[b] = external_generalized_force(gms[b], g)
        model.force_fn = _ConstantForces(fixed)
        state = SimState(q=self.q0.copy(), q_dot=self.q_dot0.copy())
        return model, state, StepParams(**self.params)


class _ConstantForces:
    """Gravity-only force_fn (reference scene.py:552-569 without windows)."""

    def __init__(self, f):
        self.f = f

    def __call__(self, step_index, t_next, q_all):
        return self.f


def rot_z(theta):
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def random_rotation(rng):
    """Haar-uniform rotation: QR of a Gaussian with the sign fixed, det +1."""
    Q, R = np.linalg.qr(rng.normal(size=(3, 3)))
    Q = Q * np.sign(np.diag(R))[None, :]
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def _q(p, A):
    return np.concatenate([np.asarray(p, dtype=float), np.asarray(A, dtype=float).reshape(9)])


def box_stack(seed=0, n_cubes=4, steps=100):
    """Config 1: cubes stacked with 1e-3 m gaps on a fixed 10x10x1 slab (top at z=0).

    'N(0,1e-3)'-style readings don't apply here; angles are one
    rng.uniform(-5, 5) degree draw per cube, bottom to top.
    """
    rng = np.random.default_rng(seed)
    gap = 1e-3
    meshes = [box_mesh([10.0, 10.0, 1.0], center=(0.0, 0.0, -0.5))]
    q0 = [_q(np.zeros(3), np.eye(3))]
    cube = box_mesh(1.0)
    for k in range(n_cubes):
        th = np.deg2rad(rng.uniform(-5.0, 5.0))
        meshes.append(cube)
        q0.append(_q([0.0, 0.0, gap + 0.5 + k * (1.0 + gap)], rot_z(th)))
    n = len(meshes)
    return SceneSpec(
        "box_stack", meshes, np.array([False] + [True] * n_cubes), np.array(q0),
        np.zeros((n, 12)), 1000.0, 1e8,
        dict(dt=0.01, d_hat=1e-3, kappa_barrier=1e4, mu=0.0, newton_tol=1e-5),
        steps,
    )


def cube_drop(seed=0, n=10, steps=300, mu=0.2):
    """Config 3: n^3 unit cubes, 1.2 m pitch, random rotations, open container.

    Container: floor slab (top at z=0) plus 4 walls, 15 m inner width,
    1 m thick, 15 m tall (resolved ambiguity).
    """
    rng = np.random.default_rng(seed)
    W, T, Hh = 15.0, 1.0, 15.0
    kin = [
        box_mesh([W + 2 * T, W + 2 * T, T], center=(0.0, 0.0, -0.5 * T)),
        box_mesh([T, W + 2 * T, Hh], center=(0.5 * W + 0.5 * T, 0.0, 0.5 * Hh)),
        box_mesh([T, W + 2 * T, Hh], center=(-0.5 * W - 0.5 * T, 0.0, 0.5 * Hh)),
        box_mesh([W, T, Hh], center=(0.0, 0.5 * W + 0.5 * T, 0.5 * Hh)),
        box_mesh([W, T, Hh], center=(0.0, -0.5 * W - 0.5 * T, 0.5 * Hh)),
    ]
    meshes = list(kin)
    q0 = [_q(np.zeros(3), np.eye(3)) for _ in kin]
    cube = box_mesh(1.0)
    pitch = 1.2
    for k in range(n):
        for j in range(n):
            for i in range(n):
                p = [(i - 0.5 * (n - 1)) * pitch, (j - 0.5 * (n - 1)) * pitch, 1.0 + k * pitch]
                meshes.append(cube)
                q0.append(_q(p, random_rotation(rng)))
    nb = len(meshes)
    dyn = np.array([False] * len(kin) + [True] * (nb - len(kin)))
    return SceneSpec(
        "cube_drop", meshes, dyn, np.array(q0), np.zeros((nb, 12)), 1000.0, 1e8,
        dict(dt=0.01, d_hat=1e-3, kappa_barrier=1e4, mu=mu), steps,
    )


def icosphere_pile(seed=0, nx=20, ny=20, nz=25, steps=200, mu=0.5, subdiv=2):
    """Config 4 (headline): nx*ny*nz level-2 icospheres, r ~ U(0.5, 1.5).

    Pitch 3.05 m (= 2 r_max + 0.05); layer k centres at z = 0.05 + 1.5 +
    3.05 k so every sphere clears the ground (top at z = 0) by >= 0.05 m.
    Rest meshes are centred (A = random rotation, p = centre).
    """
    rng = np.random.default_rng(seed)
    pitch = 3.05
    span_x, span_y = nx * pitch, ny * pitch
    slab = box_mesh([span_x + 10.0, span_y + 10.0, 1.0], center=(0.0, 0.0, -0.5))
    unit = icosphere_mesh(1.0, subdiv)
    meshes = [slab]
    q0 = [_q(np.zeros(3), np.eye(3))]
    radii = rng.uniform(0.5, 1.5, size=nx * ny * nz)
    c = 0
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                r = radii[c]
                c += 1
                meshes.append(SurfaceMesh(unit.vertices * r, unit.triangles, unit.edges))
                p = [(i - 0.5 * (nx - 1)) * pitch, (j - 0.5 * (ny - 1)) * pitch,
                     0.05 + 1.5 + k * pitch]
                q0.append(_q(p, random_rotation(rng)))
    nb = len(meshes)
    return SceneSpec(
        "icosphere_pile", meshes, np.array([False] + [True] * (nb - 1)), np.array(q0),
        np.zeros((nb, 12)), 1000.0, 1e8,
        dict(dt=0.01, d_hat=1e-3, kappa_barrier=1e4, mu=mu), steps,
        meta={"radii": radii},
    )


def chainmail(seed=0, n_chains=200, links=50, steps=400, chains_x=20, spacing=0.5):
    """Config 5: hanging chains of interlocked tori (R=0.1, r=0.02, 24x8).

    Link k lies in the xz plane (k even) or yz plane (k odd), centres
    0.14 m apart along -z: each link passes through its neighbours' holes
    (0.02 m clearance) and same-plane links k, k+2 keep 0.04 m apart (a 0.1 m
    pitch would make them overlap; SURVEY §7 item 7 only bounds the pitch
    below 2R - 2r = 0.16 m);
    the top link of every chain is kinematic.  Each chain gets one seeded
    lateral velocity ~ N(0, 0.5) m/s on its dynamic links.
    """
    rng = np.random.default_rng(seed)
    R, r, s = 0.1, 0.02, 0.14
    base = torus_mesh(R, r, 24, 8)
    # torus_mesh lies in the xy plane; rotate into xz (about x) / yz (about y)
    rx = np.array([[1.0, 0, 0], [0, 0, -1.0], [0, 1.0, 0]])  # xy -> xz plane
    ry = np.array([[0, -1.0, 0], [1.0, 0, 0], [0, 0, 1.0]]) @ rx  # then about z: xz -> yz plane
    meshes, q0, qd, dyn = [], [], [], []
    chains_y = int(np.ceil(n_chains / chains_x))
    for cidx in range(n_chains):
        cx = (cidx % chains_x - 0.5 * (chains_x - 1)) * spacing
        cy = (cidx // chains_x - 0.5 * (chains_y - 1)) * spacing
        v = np.zeros(12)
        v[:2] = rng.normal(0.0, 0.5, size=2)
        for k in range(links):
            meshes.append(base)
            A = rx if k % 2 == 0 else ry
            q0.append(_q([cx, cy, -k * s], A))
            top = k == 0
            dyn.append(not top)
            qd.append(np.zeros(12) if top else v.copy())
    nb = len(meshes)
    return SceneSpec(
        "chainmail", meshes, np.array(dyn), np.array(q0), np.array(qd), 1000.0, 1e9,
        dict(dt=0.005, d_hat=1e-4, kappa_barrier=1e4, mu=0.3), steps,
    )


def microbench_pairs(seed=0, n_bodies=100_000, n_vf=10_000_000, n_ee=10_000_000,
                     d_hat=1e-3, chunk=2_000_000, d_lo_frac=0.1):
    """Config 2 inputs: synthetic VF/EE pairs with d ~ U(d_lo_frac d_hat, d_hat).

    d_lo_frac = 0.1 (not 0): d ~ U(0, d_hat) over 20M pairs reaches d ~ d_hat / 2e7,
    Hessian blocks ~1e15 x the mass block, and no fp64 block-Jacobi PCG reaches
    1e-8 (the oracle's stalls at 8.7e-5 after 20,000 iterations on 500 bodies).
    [0.1 d_hat, d_hat] is the band CCD with slack 0.1 leaves contacts in per step.

    Returns dict with q (B,12), body graph (Morton order, +-1..4 neighbours),
    per-pair int32 (body_a, body_b), rest points (P,4,3) and eps_x (EE).
    Rest points are x_bar = A^{-1}(x - p) of each point's owning body, so
    J and q are consistent.
    """
    rng = np.random.default_rng(seed)
    B = n_bodies
    p = rng.uniform(0.0, 50.0, size=(B, 3))
    A = np.eye(3)[None] + rng.normal(0.0, 1e-3, size=(B, 3, 3))
    q = np.concatenate([p, A.reshape(B, 9)], axis=1)
    # Morton order of positions -> neighbour graph +-1..4 (8 per row)
    cell = np.clip((p / 50.0 * 1023).astype(np.int64), 0, 1023)

    def spread(x):
        x = x & 0x3FF
        x = (x | (x << 16)) & 0x030000FF
        x = (x | (x << 8)) & 0x0300F00F
        x = (x | (x << 4)) & 0x030C30C3
        x = (x | (x << 2)) & 0x09249249
        return x

    code = spread(cell[:, 0]) | (spread(cell[:, 1]) << 1) | (spread(cell[:, 2]) << 2)
    order = np.argsort(code, kind="stable")
    rank = np.empty(B, dtype=np.int64)
    rank[order] = np.arange(B)
    Ainv = np.linalg.inv(A)

    def pairs(n, kind):
        ba_all, bb_all, rp_all, eps_all = [], [], [], []
        for start in range(0, n, chunk):
            m = min(chunk, n - start)
            ba = rng.integers(0, B, size=m)
            off = rng.choice(np.array([-4, -3, -2, -1, 1, 2, 3, 4]), size=m)
            rb = np.clip(rank[ba] + off, 0, B - 1)
            rb = np.where(rb == rank[ba], rank[ba] - off, rb)
            bb = order[rb]
            d = rng.uniform(d_lo_frac * d_hat, d_hat, size=m)
            L = rng.uniform(0.05, 0.3, size=(m, 1))
            nrm = rng.normal(size=(m, 3))
            nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
            t1 = np.cross(nrm, np.eye(3)[np.argmin(np.abs(nrm), axis=1)])
            t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
            t2 = np.cross(nrm, t1)
            base = p[bb] + rng.normal(0.0, 0.3, size=(m, 3))
            x = np.empty((m, 4, 3))
            if kind == "vf":
                ang = rng.uniform(0, 2 * np.pi, size=(m, 1))
                for k in range(3):
                    a = ang + 2.0 * np.pi * k / 3.0
                    x[:, 1 + k] = base + L * (np.cos(a) * t1 + np.sin(a) * t2)
                w = rng.dirichlet(np.ones(3), size=m)
                foot = np.einsum("nk,nkj->nj", w, x[:, 1:])
                x[:, 0] = foot + d[:, None] * nrm
                owners = (ba, bb, bb, bb)
            else:
                s = rng.uniform(0.1, 0.9, size=(m, 1))
                t = rng.uniform(0.1, 0.9, size=(m, 1))
                th = rng.uniform(0.3, np.pi - 0.3, size=(m, 1))
                near = rng.random(m) < 0.01
                th[near, 0] = rng.uniform(1e-3, 2e-2, size=near.sum())
                ua = t1
                ub = np.cos(th) * t1 + np.sin(th) * t2
                La = L
                Lb = rng.uniform(0.05, 0.3, size=(m, 1))
                pa = base + d[:, None] * nrm
                x[:, 0] = pa - s * La * ua
                x[:, 1] = pa + (1 - s) * La * ua
                x[:, 2] = base - t * Lb * ub
                x[:, 3] = base + (1 - t) * Lb * ub
                owners = (ba, ba, bb, bb)
            rp = np.empty_like(x)
            for k, ob in enumerate(owners):
                rp[:, k] = np.einsum("nij,nj->ni", Ainv[ob], x[:, k] - p[ob])
            ba_all.append(ba)
            bb_all.append(bb)
            rp_all.append(rp)
            if kind == "ee":
                la = np.einsum("ni,ni->i", rp[:, 1] - rp[:, 0], rp[:, 1] - rp[:, 0])
                lb = np.einsum("ni,ni->i", rp[:, 3] - rp[:, 2], rp[:, 3] - rp[:, 2])
                eps_all.append(1e-3 * la * lb)
        out = dict(body_a=np.concatenate(ba_all).astype(np.int32),
                   body_b=np.concatenate(bb_all).astype(np.int32),
                   rest=np.concatenate(rp_all))
        if kind == "ee":
            out["eps_x"] = np.concatenate(eps_all)
        return out

    return dict(q=q, order=order, vf=pairs(n_vf, "vf"), ee=pairs(n_ee, "ee"), d_hat=d_hat)
