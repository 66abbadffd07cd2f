"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain-numpy restatement of the reference ABD Newton step
(`stiffbody`, /root/reference/pkg/src/stiffbody/*.py) used solely as the
checker by `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py`.  The product path
(`paper_2201_10022_b200`) never imports this module; it runs the sm_100a
kernels in `paper_2201_10022_b200/csrc` and fails loudly without them.

Pinning: every function here is checked against golden vectors produced by
running the reference itself on seeded inputs (`tests/golden/make_golden.py`
-> `tests/golden/*.npz`, checked in `tests/test_oracle_golden.py`).

Inputs are plain arrays / duck-typed body records with the attributes of
the reference `CollisionBody` (`contact.py:128-146`): rest (V,3) float,
triangles (T,3) int, edges (E,2) int, edge_rest_len_sq (E,), dynamic bool.
Citations are `file:line` relative to /root/reference/pkg/src/stiffbody/.
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

MOLLIFIER_SCALE = 1e-3          # distance.py:33
PARALLEL_TOL = 1e-12            # distance.py:35
ACCD_MAX_ITERS = 512            # ccd.py:23
ACCD_EPS = 1e-12                # ccd.py:26


class OracleBarrierDomainError(ValueError):
    """contact.py:53-58 — barrier at d^2 <= 0."""


class OracleStepFailure(RuntimeError):
    """solver.py:69-74 — line-search underflow."""


# ---------------------------------------------------------------------------
# small vector helpers with numpy's own reduction orders (einsum dot of
# three = (x0*y0 + x2*y2) + x1*y1 on this host; stacked gammas sequential)

def _dot3(x, y):
    return np.einsum("...i,...i->...", x, y)


def world_points(rest, q):
    """contact.py:149-153 / body.py:120-124: rest @ A^T + p."""
    q = np.asarray(q, dtype=float).reshape(12)
    return rest @ q[3:].reshape(3, 3).T + q[:3]


# ---------------------------------------------------------------------------
# closest points (distance.py:86-150, :167-204)

def pt_closest(p, t0, t1, t2):
    """Point-triangle cascade; returns (d2, region, bary). distance.py:86-150.

    Region ids: 0,1,2 vertices; 3 edge01; 4 edge12; 5 edge20; 6 interior.
    The cascade is first-match in the order VERT0, VERT1, VERT2, EDGE01,
    EDGE20, EDGE12, INTERIOR (distance.py:120-144).
    """
    p, t0, t1, t2 = (np.atleast_2d(np.asarray(v, dtype=float)) for v in (p, t0, t1, t2))
    e1 = t1 - t0
    e2 = t2 - t0
    w0, w1, w2 = p - t0, p - t1, p - t2
    d1, d2 = _dot3(e1, w0), _dot3(e2, w0)
    d3, d4 = _dot3(e1, w1), _dot3(e2, w1)
    d5, d6 = _dot3(e1, w2), _dot3(e2, w2)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    n = p.shape[0]
    zero = np.zeros(n)
    with np.errstate(divide="ignore", invalid="ignore"):
        s01 = np.where(d1 != d3, d1 / (d1 - d3), 0.0)
        s20 = np.where(d2 != d6, d2 / (d2 - d6), 0.0)
        den12 = (d4 - d3) + (d5 - d6)
        s12 = np.where(den12 != 0, (d4 - d3) / den12, 0.0)
        tot = va + vb + vc
        iv = np.where(tot != 0, vb / tot, 0.0)
        iw = np.where(tot != 0, vc / tot, 0.0)
    conds = [
        (d1 <= 0) & (d2 <= 0),
        (d3 >= 0) & (d4 <= d3),
        (d6 >= 0) & (d5 <= d6),
        (vc <= 0) & (d1 >= 0) & (d3 <= 0),
        (vb <= 0) & (d2 >= 0) & (d6 <= 0),
        (va <= 0) & (d4 - d3 >= 0) & (d5 - d6 >= 0),
    ]
    region = np.select(conds, [0, 1, 2, 3, 5, 4], default=6).astype(np.int64)
    one = np.ones(n)
    b0 = np.select(conds, [one, zero, zero, 1.0 - s01, 1.0 - s20, zero], default=1.0 - iv - iw)
    b1 = np.select(conds, [zero, one, zero, s01, zero, 1.0 - s12], default=iv)
    b2 = np.select(conds, [zero, zero, one, zero, s20, s12], default=iw)
    bary = np.stack([b0, b1, b2], axis=1)
    c = b0[:, None] * t0 + b1[:, None] * t1 + b2[:, None] * t2
    r = p - c
    return _dot3(r, r), region, bary


def ee_closest(a0, a1, b0, b1):
    """Segment-segment closest points; returns (d2, region, s, t). distance.py:167-204."""
    a0, a1, b0, b1 = (np.atleast_2d(np.asarray(v, dtype=float)) for v in (a0, a1, b0, b1))
    u = a1 - a0
    v = b1 - b0
    w = a0 - b0
    uu, vv = _dot3(u, u), _dot3(v, v)
    vw, uw, uv = _dot3(v, w), _dot3(u, w), _dot3(u, v)
    den = uu * vv - uv * uv
    par = den <= PARALLEL_TOL * uu * vv
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.clip((uv * vw - uw * vv) / np.where(den == 0, 1.0, den), 0.0, 1.0)
        s = np.where(par, 0.0, s)
        t = (uv * s + vw) / vv
        lo, hi = t <= 0.0, t >= 1.0
        t = np.clip(t, 0.0, 1.0)
        s = np.where(lo, np.clip(-uw / uu, 0.0, 1.0), s)
        s = np.where(hi, np.clip((uv - uw) / uu, 0.0, 1.0), s)
    fa = np.where(s <= 0.0, 0, np.where(s >= 1.0, 1, 2))
    fb = np.where(t <= 0.0, 0, np.where(t >= 1.0, 1, 2))
    diff = (a0 + s[:, None] * u) - (b0 + t[:, None] * v)
    return _dot3(diff, diff), (3 * fa + fb).astype(np.int64), s, t


def pair_d2(kind, z):
    z = np.asarray(z, dtype=float)
    if kind in ("vf", "vertex-face"):
        return pt_closest(z[:, 0], z[:, 1], z[:, 2], z[:, 3])[0]
    return ee_closest(z[:, 0], z[:, 1], z[:, 2], z[:, 3])[0]


# ---------------------------------------------------------------------------
# derivatives of d^2 (distance.py:238-339): envelope gradient + Schur Hessian

def _region_dirs(kind, region):
    """dgamma/dw per region, shape (N, 4, 2). distance.py:252-270."""
    n = len(region)
    D = np.zeros((n, 4, 2))
    if kind == "vf":
        e01 = np.array([0.0, 1.0, -1.0, 0.0])
        e12 = np.array([0.0, 0.0, 1.0, -1.0])
        e20 = np.array([0.0, -1.0, 0.0, 1.0])
        e_in2 = np.array([0.0, 1.0, 0.0, -1.0])
        D[region == 3, :, 0] = e01
        D[region == 4, :, 0] = e12
        D[region == 5, :, 0] = e20
        D[region == 6, :, 0] = e01
        D[region == 6, :, 1] = e_in2
    else:
        ds = np.array([-1.0, 1.0, 0.0, 0.0])
        dt = np.array([0.0, 0.0, 1.0, -1.0])
        fa, fb = region // 3, region % 3
        a_int, b_int = fa == 2, fb == 2
        D[a_int, :, 0] = ds
        D[b_int & ~a_int, :, 0] = dt
        D[b_int & a_int, :, 1] = dt
    return D


def d2_derivatives(kind, z):
    """(d2, grad (N,12), hess (N,12,12), region, gamma). distance.py:291-339."""
    z = np.asarray(z, dtype=float)
    n = len(z)
    if kind == "vf":
        d2, region, bary = pt_closest(z[:, 0], z[:, 1], z[:, 2], z[:, 3])
        gam = np.concatenate([np.ones((n, 1)), -bary], axis=1)
    else:
        d2, region, s, t = ee_closest(z[:, 0], z[:, 1], z[:, 2], z[:, 3])
        gam = np.stack([1.0 - s, s, -(1.0 - t), -t], axis=1)
    D = _region_dirs(kind, region)
    r = np.einsum("ni,nik->nk", gam, z)
    grad = 2.0 * (gam[:, :, None] * r[:, None, :]).reshape(n, 12)
    S = np.einsum("nim,nik->nkm", D, z)
    fww = 2.0 * np.einsum("nkm,nkl->nml", S, S)
    unused = ~np.any(D != 0.0, axis=1)
    fww[:, 0, 0] += unused[:, 0]
    fww[:, 1, 1] += unused[:, 1]
    F = 2.0 * (D[:, :, None, :] * r[:, None, :, None]
               + gam[:, :, None, None] * S[:, None, :, :]).reshape(n, 12, 2)
    fzz = np.zeros((n, 12, 12))
    for i in range(4):
        for j in range(4):
            fzz[:, 3 * i:3 * i + 3, 3 * j:3 * j + 3] = 2.0 * (gam[:, i] * gam[:, j])[:, None, None] * np.eye(3)
    inv = np.linalg.inv(fww)
    hess = fzz - np.einsum("nam,nml,nbl->nab", F, inv, F)
    return d2, grad, hess, region, gam


# ---------------------------------------------------------------------------
# edge-edge mollifier (distance.py:207-225, :342-401)

def ee_mollifier_value(z, eps_x):
    z = np.asarray(z, dtype=float)
    u = z[:, 1] - z[:, 0]
    v = z[:, 3] - z[:, 2]
    cr = np.cross(u, v)
    c = _dot3(cr, cr)
    eps_x = np.broadcast_to(np.asarray(eps_x, dtype=float), c.shape)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(eps_x > 0, c / eps_x, 1.0)
    return np.where(ratio >= 1.0, 1.0, ratio * (2.0 - ratio))


def ee_mollifier_derivs(z, eps_x):
    """Value, gradient (N,12), Hessian (N,12,12) of the mollifier."""
    z = np.asarray(z, dtype=float)
    n = len(z)
    u = z[:, 1] - z[:, 0]
    v = z[:, 3] - z[:, 2]
    cr = np.cross(u, v)
    c = _dot3(cr, cr)
    eps_x = np.broadcast_to(np.asarray(eps_x, dtype=float), c.shape)
    uu, vv, uv = _dot3(u, u), _dot3(v, v), _dot3(u, v)
    cu = 2.0 * (vv[:, None] * u - uv[:, None] * v)
    cv = 2.0 * (uu[:, None] * v - uv[:, None] * u)
    I3 = np.eye(3)
    huu = 2.0 * (vv[:, None, None] * I3 - v[:, :, None] * v[:, None, :])
    hvv = 2.0 * (uu[:, None, None] * I3 - u[:, :, None] * u[:, None, :])
    huv = (4.0 * u[:, :, None] * v[:, None, :] - 2.0 * v[:, :, None] * u[:, None, :]
           - 2.0 * uv[:, None, None] * I3)
    gc = np.concatenate([-cu, cu, -cv, cv], axis=1)
    sgn = (-1.0, 1.0, -1.0, 1.0)
    grp = (0, 0, 1, 1)
    hc = np.zeros((n, 12, 12))
    for i in range(4):
        for j in range(4):
            if grp[i] == 0 and grp[j] == 0:
                blk = huu
            elif grp[i] == 1 and grp[j] == 1:
                blk = hvv
            elif grp[i] == 0:
                blk = huv
            else:
                blk = np.swapaxes(huv, 1, 2)
            hc[:, 3 * i:3 * i + 3, 3 * j:3 * j + 3] = sgn[i] * sgn[j] * blk
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(eps_x > 0, c / eps_x, 1.0)
    on = ratio < 1.0
    val = np.where(on, ratio * (2.0 - ratio), 1.0)
    k1 = np.where(on, 2.0 / eps_x * (1.0 - ratio), 0.0)
    k2 = np.where(on, -2.0 / (eps_x * eps_x), 0.0)
    grad = k1[:, None] * gc
    hess = k2[:, None, None] * gc[:, :, None] * gc[:, None, :] + k1[:, None, None] * hc
    return val, grad, hess


# ---------------------------------------------------------------------------
# clamped log barrier in d^2 (contact.py:87-121)

def _domain(s):
    if np.any(s <= 0.0):
        raise OracleBarrierDomainError("barrier evaluated at non-positive squared distance")


def barrier_terms(d_sq, d_hat):
    """(B, dB/ds, d2B/ds2) with s = d^2; zero for d >= d_hat."""
    s = np.asarray(d_sq, dtype=float)
    _domain(s)
    d = np.sqrt(s)
    on = d < d_hat
    with np.errstate(divide="ignore", invalid="ignore"):
        lg = np.log(d / d_hat)
        g = d - d_hat
        b0 = -(g ** 2) * lg
        bd = -2.0 * g * lg - g ** 2 / d
        bdd = -2.0 * lg - 4.0 * g / d + g ** 2 / (d * d)
        b1 = bd / (2.0 * d)
        b2 = bdd / (4.0 * s) - bd / (4.0 * s * d)
    return np.where(on, b0, 0.0), np.where(on, b1, 0.0), np.where(on, b2, 0.0)


# ---------------------------------------------------------------------------
# gathers (contact.py:419-463) and Jacobians (contact.py:466-483)

_FLAT: dict = {}


def _flat(bodies):
    """Concatenated geometry with per-body offsets (cached per body list)."""
    key = tuple(id(b) for b in bodies)
    ent = _FLAT.get(key)
    if ent is not None:
        return ent
    vo = np.cumsum([0] + [len(b.rest) for b in bodies])
    rest = np.concatenate([b.rest for b in bodies])
    tris = np.concatenate([np.asarray(b.triangles, dtype=np.int64) + vo[i] for i, b in enumerate(bodies)])
    edges = np.concatenate([np.asarray(b.edges, dtype=np.int64) + vo[i] for i, b in enumerate(bodies)])
    to = np.cumsum([0] + [len(b.triangles) for b in bodies])
    eo = np.cumsum([0] + [len(b.edges) for b in bodies])
    el2 = np.concatenate([np.asarray(b.edge_rest_len_sq, dtype=float) for b in bodies])
    ent = (vo, to, eo, rest, tris, edges, el2)
    if len(_FLAT) > 8:
        _FLAT.clear()
    _FLAT[key] = ent
    return ent


def gather(kind, bodies, X, rows):
    """World points z (N,4,3), rest points (N,4,3), eps_x (EE) for rows (contact.py:419-463)."""
    rows = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
    vo, to, eo, rest, tris, edges, el2 = _flat(bodies)
    Xall = np.concatenate(X) if len(X) else np.zeros((0, 3))
    if kind == "vf":
        vid = np.stack([vo[rows[:, 0]] + rows[:, 1]] + [tris[to[rows[:, 2]] + rows[:, 3], k] for k in range(3)],
                       axis=1)
        eps = np.ones(len(rows))
    else:
        ea = eo[rows[:, 0]] + rows[:, 1]
        eb = eo[rows[:, 2]] + rows[:, 3]
        vid = np.stack([edges[ea, 0], edges[ea, 1], edges[eb, 0], edges[eb, 1]], axis=1)
        eps = MOLLIFIER_SCALE * el2[ea] * el2[eb]
    return Xall[vid].reshape(-1, 4, 3), rest[vid].reshape(-1, 4, 3), eps


SIDES = {"vf": (0, 1, 1, 1), "ee": (0, 0, 1, 1)}


def pair_jacobian(kind, rp):
    """(N,12,24): row 3k+a -> cols of side s_k: p_a = 1, A[a,c] = rest_k[c]."""
    n = len(rp)
    J = np.zeros((n, 12, 24))
    for k, side in enumerate(SIDES[kind]):
        o = 12 * side
        for a in range(3):
            J[:, 3 * k + a, o + a] = 1.0
            J[:, 3 * k + a, o + 3 + 3 * a:o + 6 + 3 * a] = rp[:, k]
    return J


def psd_clamp(H):
    """body.py:281-296: eigh of the symmetric part, negative eigenvalues -> 0."""
    H = np.asarray(H, dtype=float)
    Hs = 0.5 * (H + np.swapaxes(H, -1, -2))
    w, V = np.linalg.eigh(Hs)
    w = np.maximum(w, 0.0)
    return np.einsum("...ik,...k,...jk->...ij", V, w, V)


# ---------------------------------------------------------------------------
# per-pair contact terms (contact.py:486-538, :619-675)

def contact_pair_terms(kind, bodies, X, rows, kappa, d_hat):
    """Active rows plus (d2, value, g12, H12, rest points). contact.py:486-538."""
    rows = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
    z, rp, eps = gather(kind, bodies, X, rows)
    if len(rows) == 0:
        return rows, np.zeros(0), np.zeros(0), np.zeros((0, 12)), np.zeros((0, 12, 12)), rp
    keep = pair_d2(kind, z) < d_hat * d_hat
    rows, z, rp, eps = rows[keep], z[keep], rp[keep], eps[keep]
    if len(rows) == 0:
        return rows, np.zeros(0), np.zeros(0), np.zeros((0, 12)), np.zeros((0, 12, 12)), rp
    d2, gd, hd, _, _ = d2_derivatives(kind, z)
    b0, b1, b2 = barrier_terms(d2, d_hat)
    b0, b1, b2 = kappa * b0, kappa * b1, kappa * b2
    Hb = b2[:, None, None] * gd[:, :, None] * gd[:, None, :] + b1[:, None, None] * hd
    gb = b1[:, None] * gd
    if kind == "vf":
        return rows, d2, b0, gb, Hb, rp
    m, mg, mh = ee_mollifier_derivs(z, eps)
    val = m * b0
    g = mg * b0[:, None] + m[:, None] * gb
    H = (mh * b0[:, None, None] + mg[:, :, None] * gb[:, None, :]
         + gb[:, :, None] * mg[:, None, :] + m[:, None, None] * Hb)
    return rows, d2, val, g, H, rp


def kinematic_rule(g24, H24, dyn_a, dyn_b, project):
    """contact.py:619-643: project dynamic sub-block alone, zero kinematic side."""
    g24 = g24.copy()
    H24 = H24.copy()
    both = dyn_a & dyn_b
    if project and both.any():
        H24[both] = psd_clamp(H24[both])
    for mask, lo in ((dyn_a & ~dyn_b, 0), (dyn_b & ~dyn_a, 12)):
        idx = np.nonzero(mask)[0]
        if len(idx) == 0:
            continue
        sub = H24[idx][:, lo:lo + 12, lo:lo + 12]
        if project:
            sub = psd_clamp(sub)
        H24[idx] = 0.0
        H24[idx, lo:lo + 12, lo:lo + 12] = sub
        keepg = g24[idx, lo:lo + 12].copy()
        g24[idx] = 0.0
        g24[idx, lo:lo + 12] = keepg
    return g24, H24


@dataclass
class OraclePairBlocks:
    body_a: np.ndarray
    body_b: np.ndarray
    grad: np.ndarray
    hess: np.ndarray
    d_sq: np.ndarray


def _empty_blocks():
    z = np.zeros(0, dtype=np.int64)
    return OraclePairBlocks(z, z, np.zeros((0, 24)), np.zeros((0, 24, 24)), np.zeros(0))


def _cat_blocks(parts):
    parts = [p for p in parts if len(p.body_a)]
    if not parts:
        return _empty_blocks()
    return OraclePairBlocks(*(np.concatenate([getattr(p, f) for p in parts])
                              for f in ("body_a", "body_b", "grad", "hess", "d_sq")))


def all_world_points(bodies, q_all):
    q_all = np.asarray(q_all, dtype=float).reshape(len(bodies), 12)
    return [world_points(b.rest, q) for b, q in zip(bodies, q_all)]


def contact_blocks(bodies, q_all, vf, ee, kappa, d_hat, project=True):
    """contact.py:646-675."""
    X = all_world_points(bodies, q_all)
    dyn = np.array([b.dynamic for b in bodies], dtype=bool)
    out = []
    for kind, rows in (("vf", vf), ("ee", ee)):
        rows = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
        if len(rows) == 0:
            continue
        rows, d2, _, g12, H12, rp = contact_pair_terms(kind, bodies, X, rows, kappa, d_hat)
        if len(rows) == 0:
            continue
        J = pair_jacobian(kind, rp)
        g24 = np.einsum("npq,np->nq", J, g12)
        H24 = np.swapaxes(J, 1, 2) @ H12 @ J
        g24, H24 = kinematic_rule(g24, H24, dyn[rows[:, 0]], dyn[rows[:, 2]], project)
        out.append(OraclePairBlocks(rows[:, 0].copy(), rows[:, 2].copy(), g24, H24, d2))
    return _cat_blocks(out)


def contact_energy(bodies, q_all, vf, ee, kappa, d_hat):
    """contact.py:560-583."""
    X = all_world_points(bodies, q_all)
    total = 0.0
    for kind, rows in (("vf", vf), ("ee", ee)):
        rows = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
        if len(rows) == 0:
            continue
        z, _, eps = gather(kind, bodies, X, rows)
        d2 = pair_d2(kind, z)
        on = d2 < d_hat * d_hat
        if not on.any():
            continue
        b0 = kappa * barrier_terms(d2[on], d_hat)[0]
        if kind == "ee":
            b0 = ee_mollifier_value(z[on], eps[on]) * b0
        total += float(np.sum(b0))
    return total


def candidate_min_d2(bodies, q_all, vf, ee):
    """contact.py:541-557."""
    X = all_world_points(bodies, q_all)
    best = np.inf
    for kind, rows in (("vf", vf), ("ee", ee)):
        rows = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
        if len(rows):
            z, _, _ = gather(kind, bodies, X, rows)
            best = min(best, float(pair_d2(kind, z).min()))
    return None if best == np.inf else best


# ---------------------------------------------------------------------------
# lagged friction (contact.py:687-853)

@dataclass
class OracleFriction:
    body_a: np.ndarray
    body_b: np.ndarray
    lam: np.ndarray
    mu: float
    tangent_map: np.ndarray
    offset: np.ndarray
    basis: np.ndarray

    def __len__(self):
        return len(self.lam)


def _empty_friction(mu):
    z = np.zeros(0, dtype=np.int64)
    return OracleFriction(z, z, np.zeros(0), mu, np.zeros((0, 2, 24)), np.zeros((0, 2)),
                          np.zeros((0, 3, 2)))


def tangent_frames(nrm):
    """contact.py:711-719."""
    helper = np.eye(3)[np.argmin(np.abs(nrm), axis=1)]
    t1 = np.cross(nrm, helper)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(nrm, t1)
    return np.stack([t1, t2], axis=2)


def friction_precompute(bodies, q_prev, vf, ee, kappa, d_hat, mu):
    """contact.py:722-790."""
    if mu < 0:
        raise ValueError("friction coefficient must be >= 0")
    X = all_world_points(bodies, q_prev)
    qa = np.asarray(q_prev, dtype=float).reshape(len(bodies), 12)
    parts = []
    for kind, rows in (("vf", vf), ("ee", ee)):
        rows = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
        if len(rows) == 0:
            continue
        z, rp, eps = gather(kind, bodies, X, rows)
        if kind == "vf":
            d2, _, bary = pt_closest(z[:, 0], z[:, 1], z[:, 2], z[:, 3])
            gam = np.concatenate([np.ones((len(z), 1)), -bary], axis=1)
        else:
            d2, _, s, t = ee_closest(z[:, 0], z[:, 1], z[:, 2], z[:, 3])
            gam = np.stack([1.0 - s, s, -(1.0 - t), -t], axis=1)
        on = d2 < d_hat * d_hat
        if not on.any():
            continue
        rows, z, rp, gam, d2, eps = rows[on], z[on], rp[on], gam[on], d2[on], eps[on]
        d = np.sqrt(d2)
        lam = -kappa * 2.0 * d * barrier_terms(d2, d_hat)[1]
        if kind == "ee":
            lam = lam * ee_mollifier_value(z, eps)
        r = np.einsum("ni,nik->nk", gam, z)
        T = tangent_frames(r / d[:, None])
        J = pair_jacobian(kind, rp)
        Gam = np.zeros((len(rows), 3, 12))
        for k in range(4):
            Gam[:, :, 3 * k:3 * k + 3] = gam[:, k, None, None] * np.eye(3)
        tmap = np.einsum("nkm,nkp,npq->nmq", T, Gam, J)
        qp = np.concatenate([qa[rows[:, 0]], qa[rows[:, 2]]], axis=1)
        off = np.einsum("nmq,nq->nm", tmap, qp)
        parts.append(OracleFriction(rows[:, 0].copy(), rows[:, 2].copy(), lam, mu, tmap, off, T))
    if not parts:
        return _empty_friction(mu)
    return OracleFriction(*(np.concatenate([getattr(p, f) for p in parts])
                            if f != "mu" else mu
                            for f in ("body_a", "body_b", "lam", "mu", "tangent_map", "offset", "basis")))


def _f0_terms(y, eh):
    """contact.py:793-802."""
    inside = y < eh
    with np.errstate(divide="ignore", invalid="ignore"):
        f0 = np.where(inside, y * y * (1.0 - y / (3.0 * eh)) / eh + eh / 3.0, y)
        f1y = np.where(inside, 2.0 / eh - y / (eh * eh), 1.0 / np.where(y == 0, 1.0, y))
        f1p = np.where(inside, 2.0 / eh - 2.0 * y / (eh * eh), 0.0)
    return f0, f1y, f1p


def _friction_u(q_all, fr, dt, eps_v):
    qa = np.asarray(q_all, dtype=float).reshape(-1, 12)
    qp = np.concatenate([qa[fr.body_a], qa[fr.body_b]], axis=1)
    u = np.einsum("nmq,nq->nm", fr.tangent_map, qp) - fr.offset
    y = np.linalg.norm(u, axis=1)
    return (u, y) + _f0_terms(y, eps_v * dt)


def friction_energy(q_all, fr, dt, eps_v):
    """contact.py:815-820."""
    if len(fr) == 0:
        return 0.0
    f0 = _friction_u(q_all, fr, dt, eps_v)[2]
    return float(np.sum(fr.mu * fr.lam * f0))


def friction_blocks(q_all, fr, dt, eps_v, dynamic, project=True):
    """contact.py:823-853."""
    if len(fr) == 0:
        return _empty_blocks()
    u, y, _, f1y, f1p = _friction_u(q_all, fr, dt, eps_v)
    sc = fr.mu * fr.lam
    gu = sc[:, None] * f1y[:, None] * u
    with np.errstate(divide="ignore", invalid="ignore"):
        an = np.where(y > 0, (f1p - f1y) / np.where(y == 0, 1.0, y * y), 0.0)
    Hu = sc[:, None, None] * (f1y[:, None, None] * np.eye(2) + an[:, None, None] * u[:, :, None] * u[:, None, :])
    if project:
        Hu = psd_clamp(Hu)
    G = fr.tangent_map
    g24 = np.einsum("nmq,nm->nq", G, gu)
    H24 = np.einsum("nmq,nml,nlr->nqr", G, Hu, G)
    dynamic = np.asarray(dynamic, dtype=bool)
    g24, H24 = kinematic_rule(g24, H24, dynamic[fr.body_a], dynamic[fr.body_b], project=False)
    return OraclePairBlocks(fr.body_a.copy(), fr.body_b.copy(), g24, H24, np.full(len(fr), np.inf))


# ---------------------------------------------------------------------------
# orthogonality potential (body.py:229-278)

def ortho_energy(q, k):
    A = np.asarray(q, dtype=float).reshape(12)[3:].reshape(3, 3)
    G = A @ A.T
    E = G - np.eye(3)
    return k * float(np.sum(np.diag(E) ** 2) + np.sum((G - np.diag(np.diag(G))) ** 2))


def ortho_gradient(q, k):
    A = np.asarray(q, dtype=float).reshape(12)[3:].reshape(3, 3)
    out = np.zeros(12)
    out[3:] = (4.0 * k) * ((A @ A.T - np.eye(3)) @ A).reshape(9)
    return out


def ortho_hessian(q, k):
    A = np.asarray(q, dtype=float).reshape(12)[3:].reshape(3, 3)
    G = A @ A.T
    s = 4.0 * k
    S = A.T @ A  # sum_i a_i a_i^T
    H = np.zeros((12, 12))
    for i in range(3):
        ai = A[i]
        for j in range(3):
            if i == j:
                blk = 2.0 * np.outer(ai, ai) + (G[i, i] - 1.0) * np.eye(3) + (S - np.outer(ai, ai))
            else:
                blk = np.outer(A[j], ai) + G[i, j] * np.eye(3)
            H[3 + 3 * i:6 + 3 * i, 3 + 3 * j:6 + 3 * j] = s * blk
    return H


def ortho_error(q):
    A = np.asarray(q, dtype=float).reshape(12)[3:].reshape(3, 3)
    return float(np.linalg.norm(A @ A.T - np.eye(3)))


# ---------------------------------------------------------------------------
# broad phase (contact.py:338-412), restated as its exact set:
# every kind-compatible inter-body primitive pair, in body pairs with >= 1
# dynamic body, whose closed d_hat/2-inflated swept boxes overlap.

def _prim_boxes(body, X0, X1, h):
    vlo = np.minimum(X0, X1) - h
    vhi = np.maximum(X0, X1) + h
    e, t = body.edges, body.triangles
    elo = np.minimum(vlo[e[:, 0]], vlo[e[:, 1]])
    ehi = np.maximum(vhi[e[:, 0]], vhi[e[:, 1]])
    tlo = np.minimum(np.minimum(vlo[t[:, 0]], vlo[t[:, 1]]), vlo[t[:, 2]])
    thi = np.maximum(np.maximum(vhi[t[:, 0]], vhi[t[:, 1]]), vhi[t[:, 2]])
    return (vlo, vhi), (elo, ehi), (tlo, thi)


def _box_hits(alo, ahi, blo, bhi):
    if len(alo) == 0 or len(blo) == 0:
        return np.zeros((0, 2), dtype=np.int64)
    hit = np.all((alo[:, None, :] <= bhi[None, :, :]) & (blo[None, :, :] <= ahi[:, None, :]), axis=2)
    return np.argwhere(hit).astype(np.int64)


def _clip(lo, hi, olo, ohi):
    return np.nonzero(np.all((lo <= ohi) & (olo <= hi), axis=1))[0]


def _lexsort_rows(rows):
    if len(rows) == 0:
        return np.zeros((0, 4), dtype=np.int64)
    rows = np.asarray(rows, dtype=np.int64)
    return rows[np.lexsort((rows[:, 3], rows[:, 1], rows[:, 2], rows[:, 0]))]


@dataclass
class OracleCandidates:
    vf: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), dtype=np.int64))
    ee: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), dtype=np.int64))
    overlap_pairs: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), dtype=np.int64))

    def __len__(self):
        return len(self.vf) + len(self.ee)


_BP = {}  # per-call inputs shared with forked workers


def _bp_pairs(lo_hi):
    """Primitive candidates of the overlapping body pairs pairs[lo:hi] (contact.py:276-335)."""
    boxes, blo, bhi, pairs = _BP["boxes"], _BP["blo"], _BP["bhi"], _BP["pairs"]
    vf, ee = [], []
    for i, j in pairs[lo_hi[0]:lo_hi[1]]:
        i, j = int(i), int(j)
        olo, ohi = np.maximum(blo[i], blo[j]), np.minimum(bhi[i], bhi[j])
        sel = []
        for bx in (boxes[i], boxes[j]):
            sel.append([(_clip(lo, hi, olo, ohi), lo, hi) for lo, hi in bx])
        (vi, vlo_i, vhi_i), (ei, elo_i, ehi_i), (ti, tlo_i, thi_i) = sel[0]
        (vj, vlo_j, vhi_j), (ej, elo_j, ehi_j), (tj, tlo_j, thi_j) = sel[1]
        for (a_idx, alo, ahi, b_idx, blo_, bhi_, ba, bb, kind) in (
            (vi, vlo_i, vhi_i, tj, tlo_j, thi_j, i, j, "vf"),
            (vj, vlo_j, vhi_j, ti, tlo_i, thi_i, j, i, "vf"),
            (ei, elo_i, ehi_i, ej, elo_j, ehi_j, i, j, "ee"),
        ):
            hit = _box_hits(alo[a_idx], ahi[a_idx], blo_[b_idx], bhi_[b_idx])
            if len(hit) == 0:
                continue
            rows = np.empty((len(hit), 4), dtype=np.int64)
            rows[:, 0], rows[:, 1] = ba, a_idx[hit[:, 0]]
            rows[:, 2], rows[:, 3] = bb, b_idx[hit[:, 1]]
            (vf if kind == "vf" else ee).append(rows)
    z = np.zeros((0, 4), dtype=np.int64)
    return (np.concatenate(vf) if vf else z), (np.concatenate(ee) if ee else z)


def broad_phase(bodies, q_start, q_end, d_hat, workers=1):
    """contact.py:338-412: exact candidate set, sorted by (c0, c2, c1, c3).  The body
    pairs are independent, so `workers` > 1 splits them over forked processes (the
    result is the same set; rows are sorted afterwards)."""
    n = len(bodies)
    h = 0.5 * d_hat
    X0 = all_world_points(bodies, q_start)
    X1 = all_world_points(bodies, q_end)
    boxes = [_prim_boxes(b, x0, x1, h) for b, x0, x1 in zip(bodies, X0, X1)]
    blo = np.array([bx[0][0].min(axis=0) for bx in boxes]).reshape(n, 3)
    bhi = np.array([bx[0][1].max(axis=0) for bx in boxes]).reshape(n, 3)
    dyn = np.array([b.dynamic for b in bodies], dtype=bool)
    # body pairs i < j with a dynamic side and closed box overlap (contact.py:366-369),
    # tested in row chunks; listed in (i, j) lexicographic order
    pairs = []
    for i0 in range(0, n, 256):
        i1 = min(n, i0 + 256)
        hit = np.all((blo[i0:i1, None, :] <= bhi[None, :, :]) & (blo[None, :, :] <= bhi[i0:i1, None, :]), axis=2)
        hit &= np.arange(n)[None, :] > np.arange(i0, i1)[:, None]
        hit &= dyn[i0:i1, None] | dyn[None, :]
        ii, jj = np.nonzero(hit)
        pairs.append(np.stack([ii + i0, jj], axis=1))
    pairs = np.concatenate(pairs).astype(np.int64) if pairs else np.zeros((0, 2), dtype=np.int64)
    _BP.update(boxes=boxes, blo=blo, bhi=bhi, pairs=pairs)
    try:
        if workers > 1 and len(pairs) > 64:
            import multiprocessing as mp

            cuts = np.linspace(0, len(pairs), 4 * workers + 1).astype(int)
            with mp.get_context("fork").Pool(workers) as pool:
                parts = pool.map(_bp_pairs, list(zip(cuts[:-1], cuts[1:])))
        else:
            parts = [_bp_pairs((0, len(pairs)))]
    finally:
        _BP.clear()
    vf = [p[0] for p in parts if len(p[0])]
    ee = [p[1] for p in parts if len(p[1])]
    return OracleCandidates(
        _lexsort_rows(np.concatenate(vf)) if vf else np.zeros((0, 4), dtype=np.int64),
        _lexsort_rows(np.concatenate(ee)) if ee else np.zeros((0, 4), dtype=np.int64),
        pairs.reshape(-1, 2),
    )


# ---------------------------------------------------------------------------
# ACCD (ccd.py:59-153)

def accd(kind, x, dx, slack=0.1, t_max=1.0, max_iters=ACCD_MAX_ITERS):
    """Additive CCD conservative advancement. ccd.py:59-104."""
    x = np.array(x, dtype=float, copy=True).reshape(-1, 4, 3)
    dx = np.asarray(dx, dtype=float).reshape(-1, 4, 3)
    n = len(x)
    if n == 0:
        return np.zeros(0)
    k = "vf" if kind in ("vf", "vertex-face") else "ee"
    p = dx - dx.mean(axis=1, keepdims=True)
    nm = np.linalg.norm(p, axis=2)
    if k == "vf":
        lp = nm[:, 0] + nm[:, 1:].max(axis=1)
    else:
        lp = nm[:, :2].max(axis=1) + nm[:, 2:].max(axis=1)
    d0s = pair_d2(k, x)
    if np.any(d0s <= 0.0):
        raise ValueError("CCD query issued at non-positive initial distance")
    d0 = np.sqrt(d0s)
    gap = slack * d0
    t = np.zeros(n)
    live = lp > 0.0
    t[~live] = t_max
    for _ in range(max_iters):
        if not live.any():
            break
        idx = np.nonzero(live)[0]
        d = np.sqrt(pair_d2(k, x[idx]))
        adv = d - gap[idx]
        stall = adv < ACCD_EPS * d0[idx]
        tl = np.where(stall, 0.0, adv / lp[idx])
        tn = t[idx] + tl
        done = tn >= t_max
        t[idx] = np.where(done, t_max, tn)
        x[idx] += np.where(done, 0.0, tl)[:, None, None] * p[idx]
        live[idx[stall | done]] = False
    return np.minimum(t, t_max)


def step_filter(bodies, q_all, dq, vf, ee, slack=0.1):
    """ccd.py:119-153."""
    X = all_world_points(bodies, q_all)
    dqa = np.asarray(dq, dtype=float).reshape(len(bodies), 12)
    D = [world_points(b.rest, d) if b.dynamic else np.zeros_like(b.rest) for b, d in zip(bodies, dqa)]
    alpha = 1.0
    for kind, rows in (("vf", vf), ("ee", ee)):
        rows = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
        if len(rows) == 0:
            continue
        z, _, _ = gather(kind, bodies, X, rows)
        dz, _, _ = gather(kind, bodies, D, rows)
        alpha = min(alpha, float(accd(kind, z, dz, slack, 1.0).min()))
    return alpha


# ---------------------------------------------------------------------------
# incremental potential, assembly, solve, line search, Newton step
# (solver.py:179-628)

@dataclass
class OracleModel:
    bodies: list
    mass: list            # 12x12 matrices (None for kinematic)
    stiffness: list       # kappa_ortho * volume (None for kinematic)

    def __post_init__(self):
        self.dynamic = np.array([b.dynamic for b in self.bodies], dtype=bool)
        self.dyn = np.nonzero(self.dynamic)[0]
        self.slot = np.full(len(self.bodies), -1, dtype=np.int64)
        self.slot[self.dyn] = np.arange(len(self.dyn))


@dataclass
class OracleParams:
    dt: float
    d_hat: float = 1e-3
    kappa_barrier: float = 1e4
    mu: float = 0.0
    epsilon_v: float = 1e-3
    newton_tol: float = 1e-2
    max_newton_iters: int = 64
    ccd_slack: float = 0.1
    ccd_step_scale: float = 0.9


@dataclass
class OracleIP:
    q_tilde: np.ndarray
    friction: OracleFriction
    cands: OracleCandidates


def q_tilde(model, q, q_dot, forces, dt):
    """solver.py:179-190."""
    out = np.array(q, dtype=float, copy=True)
    for b in model.dyn:
        out[b] = q[b] + dt * q_dot[b] + dt ** 2 * np.linalg.solve(model.mass[b], forces[b])
    return out


def ip_value(model, q_all, ip, prm):
    """solver.py:193-205."""
    e = 0.0
    for b in model.dyn:
        d = q_all[b] - ip.q_tilde[b]
        e += 0.5 * float(d @ model.mass[b] @ d)
        e += prm.dt ** 2 * ortho_energy(q_all[b], model.stiffness[b])
    e += contact_energy(model.bodies, q_all, ip.cands.vf, ip.cands.ee, prm.kappa_barrier, prm.d_hat)
    e += friction_energy(q_all, ip.friction, prm.dt, prm.epsilon_v)
    return e


def assemble(model, q_all, ip, prm):
    """solver.py:257-342.  Returns (grad (n_dyn*12,), diag (n,12,12), off dict)."""
    n = len(model.dyn)
    grad = np.zeros((n, 12))
    diag = np.zeros((n, 12, 12))
    keys = set()
    srcs = [ip.cands.overlap_pairs]
    if len(ip.friction):
        srcs.append(np.stack([ip.friction.body_a, ip.friction.body_b], axis=1))
    for arr in srcs:
        for i, j in np.asarray(arr).reshape(-1, 2):
            si, sj = model.slot[i], model.slot[j]
            if si >= 0 and sj >= 0:
                keys.add((min(si, sj), max(si, sj)))
    off = {k: np.zeros((12, 12)) for k in sorted(keys)}
    oh = np.zeros((max(n, 1), 12, 12))
    for b in model.dyn:
        s = model.slot[b]
        grad[s] += model.mass[b] @ (q_all[b] - ip.q_tilde[b])
        grad[s] += prm.dt ** 2 * ortho_gradient(q_all[b], model.stiffness[b])
        diag[s] += model.mass[b]
        oh[s] = ortho_hessian(q_all[b], model.stiffness[b])
    if n:
        diag += prm.dt ** 2 * psd_clamp(oh[:n])
    parts = [contact_blocks(model.bodies, q_all, ip.cands.vf, ip.cands.ee, prm.kappa_barrier, prm.d_hat),
             friction_blocks(q_all, ip.friction, prm.dt, prm.epsilon_v, model.dynamic)]
    for blk in parts:
        for k in range(len(blk.body_a)):
            sa, sb = model.slot[blk.body_a[k]], model.slot[blk.body_b[k]]
            if sa >= 0:
                grad[sa] += blk.grad[k, :12]
                diag[sa] += blk.hess[k, :12, :12]
            if sb >= 0:
                grad[sb] += blk.grad[k, 12:]
                diag[sb] += blk.hess[k, 12:, 12:]
            if sa >= 0 and sb >= 0:
                up = blk.hess[k, :12, 12:]
                off[(min(sa, sb), max(sa, sb))] += up if sa < sb else up.T
    return grad.reshape(-1), diag, off


def bsr_dense(diag, off):
    n = len(diag)
    A = np.zeros((12 * n, 12 * n))
    for i in range(n):
        A[12 * i:12 * i + 12, 12 * i:12 * i + 12] = diag[i]
    for (i, j), B in off.items():
        A[12 * i:12 * i + 12, 12 * j:12 * j + 12] = B
        A[12 * j:12 * j + 12, 12 * i:12 * i + 12] = B.T
    return A


def bsr_matvec(diag, off, x):
    """sparse.py:77-84."""
    xb = x.reshape(len(diag), 12)
    y = np.einsum("nij,nj->ni", diag, xb)
    for (i, j), B in off.items():
        y[i] += B @ xb[j]
        y[j] += B.T @ xb[i]
    return y.reshape(-1)


def solve_dense(diag, off, g):
    """Newton solve H dq = -g (dense Cholesky stands in for sparse.py:90-161)."""
    if len(diag) == 0:
        return np.zeros(0)
    A = bsr_dense(diag, off)
    L = np.linalg.cholesky(0.5 * (A + A.T))
    return -np.linalg.solve(L.T, np.linalg.solve(L, g))


def bsr_csr(diag, off):
    """The full symmetric BSR (both triangles) as a scipy CSR matrix."""
    import scipy.sparse as sp

    n = len(diag)
    keys = list(off.keys())
    rows = [np.arange(n)] + ([np.array([k[0] for k in keys]), np.array([k[1] for k in keys])] if keys else [])
    cols = [np.arange(n)] + ([np.array([k[1] for k in keys]), np.array([k[0] for k in keys])] if keys else [])
    blks = [diag] + ([np.array([off[k] for k in keys]), np.array([off[k].T for k in keys])] if keys else [])
    r, c, b = np.concatenate(rows), np.concatenate(cols), np.concatenate(blks)
    ii = (12 * r[:, None, None] + np.arange(12)[None, :, None]).repeat(12, axis=2)
    jj = (12 * c[:, None, None] + np.arange(12)[None, None, :]).repeat(12, axis=1)
    return sp.csr_matrix((b.reshape(-1), (ii.reshape(-1), jj.reshape(-1))), shape=(12 * n, 12 * n))


def solve_sparse(diag, off, g, rel_tol=1e-8, max_refine=3):
    """Newton solve H dq = -g by a sparse direct factorisation (SuperLU) with the
    refinement contract of BlockCholesky.solve_refined (sparse.py:90-161): the
    reference's algorithm class at scenes where a dense matrix cannot be formed."""
    from scipy.sparse.linalg import splu

    if len(diag) == 0:
        return np.zeros(0)
    A = bsr_csr(diag, off).tocsc()
    lu = splu(A)
    b = -np.asarray(g, dtype=float)
    x = lu.solve(b)
    bn = np.linalg.norm(b)
    for _ in range(max_refine):
        r = b - A @ x
        if np.linalg.norm(r) <= rel_tol * bn:
            break
        x = x + lu.solve(r)
    return x


def pcg_block_jacobi(diag, off, b, rel_tol=1e-8, max_iters=100000):
    """numpy block-Jacobi PCG (CPU baseline for the sm_100a PCG)."""
    n = len(diag)
    Minv = np.linalg.inv(diag)
    x = np.zeros(12 * n)
    r = b.copy()
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return x, 0
    z = np.einsum("nij,nj->ni", Minv, r.reshape(n, 12)).reshape(-1)
    p = z.copy()
    rz = r @ z
    for it in range(1, max_iters + 1):
        Ap = bsr_matvec(diag, off, p)
        a = rz / (p @ Ap)
        x += a * p
        r -= a * Ap
        if np.linalg.norm(r) <= rel_tol * bn:
            return x, it
        z = np.einsum("nij,nj->ni", Minv, r.reshape(n, 12)).reshape(-1)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, max_iters


def line_search(model, q_all, dq, ip, prm, e0=None):
    """solver.py:358-393."""
    amax = step_filter(model.bodies, q_all, dq, ip.cands.vf, ip.cands.ee, prm.ccd_slack)
    alpha = 1.0 if amax >= 1.0 else min(1.0, prm.ccd_step_scale * amax)
    if e0 is None:
        e0 = ip_value(model, q_all, ip, prm)
    while True:
        e = ip_value(model, q_all + alpha * dq, ip, prm)
        if e < e0:
            return alpha, e, amax
        alpha *= 0.5
        if alpha < 1e-12:
            raise OracleStepFailure("line search underflow")


def global_min_distance(bodies, q_all):
    """solver.py:396-473 restated: body pairs in ascending box-gap order with an
    early exit once the gap reaches the best distance (solver.py:407-420);
    primitive pairs whose box gap is already >= best are skipped (exact: the
    box gap is a lower bound of the primitive distance)."""
    X = all_world_points(bodies, q_all)
    n = len(bodies)
    lo = np.array([x.min(axis=0) for x in X])
    hi = np.array([x.max(axis=0) for x in X])
    gaps = []
    for i in range(n):
        for j in range(i + 1, n):
            if not (bodies[i].dynamic or bodies[j].dynamic):
                continue
            g = np.maximum(0.0, np.maximum(lo[i] - hi[j], lo[j] - hi[i]))
            gaps.append((float(np.linalg.norm(g)), i, j))
    gaps.sort()

    def box_gap(alo, ahi, blo, bhi):
        g = np.maximum(0.0, np.maximum(alo - bhi, blo - ahi))
        return np.sqrt(np.einsum("...i,...i->...", g, g))

    best = np.inf
    for gap, i, j in gaps:
        if gap >= best:
            break
        for a, b in ((i, j), (j, i)):
            V = X[a]
            T = X[b][bodies[b].triangles]
            g = box_gap(V[:, None, :], V[:, None, :], T.min(axis=1)[None], T.max(axis=1)[None])
            vi, ti = np.nonzero(g < best)
            if len(vi):
                d2 = pt_closest(V[vi], T[ti, 0], T[ti, 1], T[ti, 2])[0]
                best = min(best, float(np.sqrt(d2.min())))
        Ea = X[i][bodies[i].edges]
        Eb = X[j][bodies[j].edges]
        g = box_gap(Ea.min(axis=1)[:, None], Ea.max(axis=1)[:, None], Eb.min(axis=1)[None], Eb.max(axis=1)[None])
        ei, ej = np.nonzero(g < best)
        if len(ei):
            d2 = ee_closest(Ea[ei, 0], Ea[ei, 1], Eb[ej, 0], Eb[ej, 1])[0]
            best = min(best, float(np.sqrt(d2.min())))
    return best


@dataclass
class OracleStepStats:
    iterations: int
    converged: bool
    min_distance: float
    candidates: int
    ip_value: float
    max_ortho_error: float
    energy_trace: list
    alphas: list
    min_iterate_distance: float = np.inf


def advance_step(model, q, q_dot, forces, prm, solver="dense", min_distance=True, audit_iterates=False):
    """solver.py:493-628 (friction_outer_iters = 1, no joint reduction); audit_iterates
    as StepParams.audit_iterates (solver.py:577-580)."""
    q0 = np.array(q, dtype=float, copy=True)
    qt = q_tilde(model, q0, q_dot, forces, prm.dt)
    cands = broad_phase(model.bodies, q0, q0, prm.d_hat)
    fr = friction_precompute(model.bodies, q0, cands.vf, cands.ee, prm.kappa_barrier, prm.d_hat, prm.mu)
    ip = OracleIP(qt, fr, cands)
    qc = q0.copy()
    iters, conv = 0, False
    trace, alphas = [], []
    min_iter = np.inf
    maxc = len(cands)
    dd = np.zeros(0)
    for _ in range(prm.max_newton_iters):
        g, D, O = assemble(model, qc, ip, prm)
        if solver == "dense":
            dd = solve_dense(D, O, g)
        elif solver == "sparse":
            dd = solve_sparse(D, O, g)
        else:
            dd = pcg_block_jacobi(D, O, -g)[0]
        if len(dd) == 0 or np.abs(dd).max() / prm.dt < prm.newton_tol:
            conv = True
            break
        if float(g @ dd) >= 0.0:
            warnings.warn("non-descent direction; steepest descent fallback", RuntimeWarning)
            dd = -g
        dq = np.zeros_like(qc)
        dq[model.dyn] = dd.reshape(-1, 12)
        ip.cands = broad_phase(model.bodies, qc, qc + dq, prm.d_hat)
        maxc = max(maxc, len(ip.cands))
        alpha, e_new, _ = line_search(model, qc, dq, ip, prm)
        qc = qc + alpha * dq
        trace.append(e_new)
        alphas.append(alpha)
        iters += 1
        if audit_iterates:
            min_iter = min(min_iter, global_min_distance(model.bodies, qc))
    if not conv:
        warnings.warn("Newton did not converge", RuntimeWarning)
    qd = np.zeros_like(qc)
    qd[model.dyn] = (qc[model.dyn] - q0[model.dyn]) / prm.dt
    md = np.nan
    if min_distance:
        cm = candidate_min_d2(model.bodies, qc, ip.cands.vf, ip.cands.ee)
        if cm is not None and cm < prm.d_hat ** 2:
            md = float(np.sqrt(cm))
        else:
            md = global_min_distance(model.bodies, qc)
    stats = OracleStepStats(
        iters, conv, md, maxc, ip_value(model, qc, ip, prm),
        max((ortho_error(qc[b]) for b in model.dyn), default=0.0), trace, alphas, min_iter)
    return qc, qd, stats


# ---------------------------------------------------------------------------
# intersection audit (intersect.py:18-42, scene.py:627-698)

def tri_intersect_batch(ta, tb):
    """Closed-triangle separating-axis test on (N,3,3) pairs (intersect.py:18-42):
    axes = face normals, 9 edge-edge crosses, 6 in-plane edge normals; an axis
    with |axis|^2 <= 1e-30 is skipped; touching counts as intersecting."""
    ta = np.asarray(ta, dtype=float).reshape(-1, 3, 3)
    tb = np.asarray(tb, dtype=float).reshape(-1, 3, 3)
    ea = np.stack([ta[:, 1] - ta[:, 0], ta[:, 2] - ta[:, 1], ta[:, 0] - ta[:, 2]], axis=1)
    eb = np.stack([tb[:, 1] - tb[:, 0], tb[:, 2] - tb[:, 1], tb[:, 0] - tb[:, 2]], axis=1)
    na = np.cross(ea[:, 0], ea[:, 1])
    nb = np.cross(eb[:, 0], eb[:, 1])
    ax = [na[:, None], nb[:, None]]
    ax += [np.cross(ea[:, i], eb[:, j])[:, None] for i in range(3) for j in range(3)]
    ax += [np.cross(ea[:, i], na)[:, None] for i in range(3)]
    ax += [np.cross(eb[:, i], nb)[:, None] for i in range(3)]
    ax = np.concatenate(ax, axis=1)
    pa = np.einsum("nak,npk->nap", ax, ta)
    pb = np.einsum("nak,npk->nap", ax, tb)
    sep = (pa.min(axis=2) > pb.max(axis=2)) | (pb.min(axis=2) > pa.max(axis=2))
    live = np.einsum("nak,nak->na", ax, ax) > 1e-30
    return ~(sep & live).any(axis=1)


def _ray_parity_inside(p, X, tris):
    """scene.py:627-649: ray along a fixed skewed direction, odd hit count = inside."""
    d = np.array([0.5424426421, 0.7866258632, 0.2954766431])
    v0, v1, v2 = X[tris[:, 0]], X[tris[:, 1]], X[tris[:, 2]]
    e1, e2 = v1 - v0, v2 - v0
    h = np.cross(np.broadcast_to(d, e2.shape), e2)
    a = np.einsum("ij,ij->i", e1, h)
    ok = np.abs(a) > 1e-14
    f = np.where(ok, 1.0 / np.where(ok, a, 1.0), 0.0)
    s = p - v0
    u = f * np.einsum("ij,ij->i", s, h)
    qv = np.cross(s, e1)
    v = f * np.einsum("ij,j->i", qv, d)
    t = f * np.einsum("ij,ij->i", e2, qv)
    return int((ok & (u >= 0) & (u <= 1) & (v >= 0) & (u + v <= 1) & (t > 1e-12)).sum()) % 2 == 1


def intersecting_body_pairs(bodies, q_all):
    """scene.py:652-698 on generalized coordinates: box-overlapping body pairs,
    triangle SAT on triangle pairs whose boxes meet the overlap box and each other,
    else containment by ray parity both ways."""
    q_all = np.asarray(q_all, dtype=float).reshape(len(bodies), 12)
    Xs = [world_points(np.asarray(b.rest, dtype=float), q_all[i]) for i, b in enumerate(bodies)]
    tris = [np.asarray(b.triangles, dtype=np.int64) for b in bodies]
    lo = [x.min(axis=0) for x in Xs]
    hi = [x.max(axis=0) for x in Xs]
    out = []
    for i in range(len(bodies)):
        for j in range(i + 1, len(bodies)):
            olo, ohi = np.maximum(lo[i], lo[j]), np.minimum(hi[i], hi[j])
            if (olo > ohi).any():
                continue
            Ta, Tb = Xs[i][tris[i]], Xs[j][tris[j]]
            alo, ahi, blo, bhi = Ta.min(axis=1), Ta.max(axis=1), Tb.min(axis=1), Tb.max(axis=1)
            ka = np.nonzero(((alo <= ohi) & (ahi >= olo)).all(axis=1))[0]
            kb = np.nonzero(((blo <= ohi) & (bhi >= olo)).all(axis=1))[0]
            hit = False
            if len(ka) and len(kb):
                m = ((alo[ka][:, None] <= bhi[kb][None]) & (blo[kb][None] <= ahi[ka][:, None])).all(axis=2)
                ii, jj = np.nonzero(m)
                hit = bool(len(ii)) and bool(tri_intersect_batch(Ta[ka[ii]], Tb[kb[jj]]).any())
            if not hit:
                hit = _ray_parity_inside(Xs[i][0], Xs[j], tris[j]) or _ray_parity_inside(Xs[j][0], Xs[i], tris[i])
            if hit:
                out.append((i, j))
    return out
