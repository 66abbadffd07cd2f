"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports `stiffbody` from /root/reference/pkg/src, evaluates it on seeded
inputs and writes tests/golden/*.npz.  The fixtures pin both the CPU oracle
(`oracle/abd_oracle.py`, CPU tests) and the sm_100a path (`-m gpu` tests);
nothing at test time reads /root/reference.
"""
from __future__ import annotations

import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import stiffbody.body as rb  # noqa: E402
import stiffbody.ccd as rccd  # noqa: E402
import stiffbody.contact as rc  # noqa: E402
import stiffbody.distance as rd  # noqa: E402
import stiffbody.mesh as rm  # noqa: E402
import stiffbody.solver as rs  # noqa: E402
import stiffbody.shapes as rshapes  # noqa: E402

from golden_io import pack_bodies, pack_offdict  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402


def save(name, d):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **d)
    print(f"wrote {name}: {os.path.getsize(path) / 1e6:.2f} MB")


# ---------------------------------------------------------------------------
def special_pt(rng):
    """Point-triangle configurations hitting every region and exact ties."""
    rows = []
    t = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    pts = [
        [0, 0, 1], [0.2, 0.2, 1], [2, 2, 0], [-1, -1, 0.3], [1.5, -0.2, 0.1], [-0.2, 1.5, -0.1],
        [0.5, -1, 0.2], [-1, 0.5, 0.2], [1, 1, 0.5], [0, 0, 0], [1, 0, 0], [0, 1, 0],
        [0.5, 0, 0], [0, 0.5, 0], [0.5, 0.5, 0], [0.25, 0.25, 0], [1.0, -0.0, 2.0], [0, 0, -3],
    ]
    for p in pts:
        rows.append(np.vstack([p, t]))
    for _ in range(400):
        rows.append(rng.normal(size=(4, 3)))
    for _ in range(200):
        tri = rng.normal(size=(3, 3))
        w = rng.dirichlet(np.ones(3))
        nrm = np.cross(tri[1] - tri[0], tri[2] - tri[0])
        nrm /= np.linalg.norm(nrm)
        rows.append(np.vstack([w @ tri + rng.uniform(-1e-3, 1e-3) * nrm, tri]))
    return np.array(rows)


def special_ee(rng):
    rows = [
        [[0, 0, 0], [1, 0, 0], [0.5, -1, 1], [0.5, 1, 1]],
        [[0, 0, 0], [1, 0, 0], [0, 0, 1], [1, 0, 1]],          # parallel
        [[0, 0, 0], [1, 0, 0], [2, 0, 1], [3, 0, 1]],          # parallel, offset
        [[0, 0, 0], [1, 0, 0], [-1, -1, 0.5], [-1, 1, 0.5]],
        [[0, 0, 0], [1, 0, 0], [1, 0, 0], [1, 1, 1]],          # shared endpoint
        [[0, 0, 0], [1, 0, 0], [0.5, 0, 0], [0.5, 0, 1]],      # touching
        [[0, 0, 0], [1, 0, 0], [0, 1e-7, 1], [1, -1e-7, 1]],   # near parallel
    ]
    rows = [np.array(r, dtype=float) for r in rows]
    for _ in range(400):
        rows.append(rng.normal(size=(4, 3)))
    for _ in range(200):
        a0 = rng.normal(size=3)
        u = rng.normal(size=3)
        v = u + rng.normal(size=3) * rng.choice([1e-1, 1e-2, 1e-3, 1e-4])
        rows.append(np.array([a0, a0 + u, a0 + rng.normal(size=3) * 0.05, a0 + rng.normal(size=3) * 0.05 + v]))
    return np.array(rows)


def gen_kernels():
    rng = np.random.default_rng(1234)
    out = {}
    zpt = special_pt(rng)
    d2, reg, bary = rd.point_triangle_closest(zpt[:, 0], zpt[:, 1], zpt[:, 2], zpt[:, 3])
    out.update(pt_z=zpt, pt_d2=d2, pt_region=reg, pt_bary=bary)
    zee = special_ee(rng)
    d2, reg, s, t = rd.edge_edge_closest(zee[:, 0], zee[:, 1], zee[:, 2], zee[:, 3])
    out.update(ee_z=zee, ee_d2=d2, ee_region=reg, ee_s=s, ee_t=t)
    # derivative kernels (non-degenerate pairs only)
    keep_pt = d2_pt = rd.point_triangle_closest(zpt[:, 0], zpt[:, 1], zpt[:, 2], zpt[:, 3])[0] > 1e-12
    zg = zpt[keep_pt]
    g = rd.pair_distance_gradients("vf", zg)
    out.update(gvf_z=zg, gvf_d2=g[0], gvf_grad=g[1], gvf_hess=g[2], gvf_region=g[3], gvf_gamma=g[4])
    keep_ee = rd.edge_edge_closest(zee[:, 0], zee[:, 1], zee[:, 2], zee[:, 3])[0] > 1e-12
    zg = zee[keep_ee]
    g = rd.pair_distance_gradients("ee", zg)
    out.update(gee_z=zg, gee_d2=g[0], gee_grad=g[1], gee_hess=g[2], gee_region=g[3], gee_gamma=g[4])
    u = zg[:, 1] - zg[:, 0]
    v = zg[:, 3] - zg[:, 2]
    eps = 1e-3 * np.einsum("ij,ij->i", u, u) * np.einsum("ij,ij->i", v, v)
    val, mg, mh = rd.ee_mollifier_grad_hess(zg, eps)
    out.update(mol_z=zg, mol_eps=eps, mol_val=val, mol_grad=mg, mol_hess=mh,
               mol_val2=rd.ee_mollifier(zg[:, 0], zg[:, 1], zg[:, 2], zg[:, 3], eps))
    # barrier
    dh = 1e-3
    ss = np.concatenate([rng.uniform(1e-14, 2 * dh * dh, 300), [dh * dh, 0.25 * dh * dh, 4 * dh * dh],
                         (dh * (1 - np.geomspace(1e-8, 1e-1, 20))) ** 2])
    out.update(bar_s=ss, bar_dhat=np.array(dh), bar_b0=rc.barrier(ss, dh),
               bar_b1=rc.barrier_d1(ss, dh), bar_b2=rc.barrier_d2(ss, dh))
    # orthogonality potential
    qs = [np.concatenate([np.zeros(3), np.eye(3).ravel()]),
          np.concatenate([np.zeros(3), np.diag([2.0, 1, 1]).ravel()])]
    for _ in range(60):
        A = scenes.random_rotation(rng) + rng.normal(0, rng.choice([1e-4, 1e-2, 0.3]), (3, 3))
        qs.append(np.concatenate([rng.normal(size=3), A.ravel()]))
    qs = np.array(qs)
    mat = rb.BodyMaterial(1000.0, 1e8, 0.37)
    out.update(
        orth_q=qs, orth_k=np.array(mat.stiffness_scale),
        orth_e=np.array([rb.ortho_energy(q, mat) for q in qs]),
        orth_g=np.array([rb.ortho_gradient(q, mat) for q in qs]),
        orth_h=np.array([rb.ortho_hessian(q, mat) for q in qs]),
        orth_hp=np.array([rb.ortho_hessian(q, mat, project_psd=True) for q in qs]),
        orth_err=np.array([rb.ortho_error(q) for q in qs]),
    )
    for k in (2, 12, 24):
        H = rng.normal(size=(40, k, k))
        out[f"psd{k}_in"] = H
        out[f"psd{k}_out"] = rb.project_psd(H)
    # ACCD
    for kind, tag in (("vertex-face", "vf"), ("edge-edge", "ee")):
        xs, dxs = [], []
        while len(xs) < 300:
            x = rng.normal(size=(4, 3))
            d2 = (rd.point_triangle_closest if tag == "vf" else rd.edge_edge_closest)(
                x[0], x[1], x[2], x[3])[0][0]
            if d2 < 1e-6:
                continue
            xs.append(x)
            dxs.append(rng.normal(size=(4, 3)) * rng.uniform(0.1, 2.0))
        xs, dxs = np.array(xs), np.array(dxs)
        dxs[:5] = dxs[:5, :1]  # common translation -> full step
        out[f"ccd_{tag}_x"] = xs
        out[f"ccd_{tag}_dx"] = dxs
        out[f"ccd_{tag}_t"] = rccd.accd_toi_batch(kind, xs, dxs, slack=0.1)
        out[f"ccd_{tag}_t3"] = rccd.accd_toi_batch(kind, xs, dxs, slack=0.3, t_max=0.7)
    save("kernels.npz", out)


# ---------------------------------------------------------------------------
def ref_bodies(meshes, dynamic):
    out = []
    for m, dyn in zip(meshes, dynamic):
        rmesh = rm.SurfaceMesh(np.array(m.vertices), np.array(m.triangles))
        assert np.array_equal(rmesh.edges, m.edges), "edge lists differ"
        out.append(rc.CollisionBody.from_mesh(rmesh, dynamic=bool(dyn)))
    return out


def ref_model(meshes, dynamic, density, kappa_o, gravity=(0, 0, -9.8)):
    bodies = ref_bodies(meshes, dynamic)
    gms, mats = [], []
    for b, m, dyn in zip(bodies, meshes, dynamic):
        if not dyn:
            gms.append(None)
            mats.append(None)
            continue
        gm, vol = rb.mass_matrix(rm.SurfaceMesh(np.array(m.vertices), np.array(m.triangles)), density)
        gms.append(gm)
        mats.append(rb.BodyMaterial(density, kappa_o, vol))
    model = rs.SystemModel(bodies, gms, mats)

    def fn(step, t, q):
        f = np.zeros((len(bodies), 12))
        for b in model.dyn_indices:
            f[b] = rb.external_generalized_force(gms[b], gravity)
        return f

    model.force_fn = fn
    return model


def contact_case(tag, meshes, dynamic, q0, dq, d_hat, kappa, mu, density, kappa_o, dt, rng, out,
                 q_dot=None):
    model = ref_model(meshes, dynamic, density, kappa_o)
    bodies = model.bodies
    n = len(bodies)
    p = f"{tag}_"
    pack_bodies(p, bodies, out)
    out[p + "q0"], out[p + "dq"] = q0, dq
    out[p + "params"] = np.array([d_hat, kappa, mu, density, kappa_o, dt])
    c0 = rc.broad_phase(bodies, q0, q0, d_hat)
    c1 = rc.broad_phase(bodies, q0, q0 + dq, d_hat)
    for nm, c in (("c0", c0), ("c1", c1)):
        out[p + nm + "_vf"], out[p + nm + "_ee"], out[p + nm + "_ov"] = c.vf, c.ee, c.overlap_pairs
    out[p + "energy"] = np.array(rc.contact_energy(bodies, q0, c0, kappa, d_hat))
    for proj in (True, False):
        blk = rc.contact_gradient_hessian(bodies, q0, c0, kappa, d_hat, project=proj)
        s = "P" if proj else "U"
        out[p + f"blk{s}_a"], out[p + f"blk{s}_b"] = blk.body_a, blk.body_b
        out[p + f"blk{s}_g"], out[p + f"blk{s}_h"], out[p + f"blk{s}_d2"] = blk.grad, blk.hess, blk.d_sq
    fr = rc.friction_precompute(bodies, q0, c0, kappa, d_hat, mu)
    out[p + "fr_a"], out[p + "fr_b"], out[p + "fr_lam"] = fr.body_a, fr.body_b, fr.lam
    out[p + "fr_tmap"], out[p + "fr_off"], out[p + "fr_basis"] = fr.tangent_map, fr.offset, fr.basis
    qp = q0.copy()
    dynm = np.array([b.dynamic for b in bodies])
    qp[dynm] += 1e-5 * rng.normal(size=(int(dynm.sum()), 12))
    out[p + "qp"] = qp
    out[p + "fr_energy"] = np.array(rc.friction_energy(qp, fr, dt, 1e-3))
    for proj in (True, False):
        fb = rc.friction_gradient_hessian(qp, fr, dt, 1e-3, dynm, project=proj)
        s = "P" if proj else "U"
        out[p + f"frb{s}_g"], out[p + f"frb{s}_h"] = fb.grad, fb.hess
    out[p + "alpha"] = np.array(rccd.step_filter(bodies, q0, dq, c1, slack=0.1))
    # assembly + IP value at a perturbed iterate with this step's IP state
    params = rs.StepParams(dt=dt, d_hat=d_hat, kappa_barrier=kappa, mu=mu)
    qd = np.zeros((n, 12)) if q_dot is None else q_dot
    state = rs.SimState(q=q0.copy(), q_dot=qd.copy())
    forces = model.forces(0, dt, q0)
    qt = rs.compute_q_tilde(model, state, params, forces)
    ip = rs.IncrementalPotentialState(q0.copy(), qd.copy(), qt, fr, c0, model)
    out[p + "qdot"], out[p + "qtilde"] = qd, qt
    g, H = rs.assemble(qp, ip, params)
    out[p + "asm_g"], out[p + "asm_diag"] = g, H.diag
    pack_offdict(p + "asm_", H.off, out)
    out[p + "ip"] = np.array(rs.ip_value(qp, ip, params))
    out[p + "masses"] = np.array([model.gmass[b].matrix if dynamic[b] else np.zeros((12, 12)) for b in range(n)])
    out[p + "stiff"] = np.array([model.materials[b].stiffness_scale if dynamic[b] else 0.0 for b in range(n)])
    dx = rs.solve_newton_system(H, g)
    out[p + "solve_dx"] = dx


def gen_contact():
    rng = np.random.default_rng(99)
    out = {}
    # two cubes, second rotated slightly; both dynamic (near-parallel edges -> mollifier)
    d_hat = 5e-2
    meshes = [rshapes.box_mesh(1.0), rshapes.box_mesh(1.0)]
    q0 = np.tile(rb.BodyCoords.identity().q, (2, 1))
    q0[1, 0] = 1.0 + d_hat / 2
    q0[1, 3:] += 0.02 * rng.normal(size=9)
    dq = np.zeros((2, 12))
    dq[1, :3] = [-0.05, 0.01, 0.0]
    dq[1, 3:] = 0.01 * rng.normal(size=9)
    contact_case("twocube", meshes, [True, True], q0, dq, d_hat, 10.0, 0.3, 1.0, 1.0, 0.01, rng, out)
    # exactly aligned cubes (parallel edges: mollifier c = 0)
    q0 = np.tile(rb.BodyCoords.identity().q, (2, 1))
    q0[1, :3] = [1.0 + 1e-2 / 3, 0.21, 0.13]
    dq = np.zeros((2, 12))
    dq[1, 0] = -0.02
    contact_case("aligned", meshes, [True, True], q0, dq, 1e-2, 1e4, 0.5, 1000.0, 1e8, 0.01, rng, out)
    # resting cube on kinematic floor (friction, kinematic sub-block rule)
    floor = rshapes.box_mesh([4.0, 4.0, 1.0], center=(0, 0, -0.5))
    cube = rshapes.box_mesh(0.5)
    q0 = np.tile(rb.BodyCoords.identity().q, (2, 1))
    q0[1, :3] = [0.3, -0.2, 0.25 + 0.4e-2]
    q0[1, 3:] = (scenes.rot_z(0.3) @ np.eye(3)).ravel() + 1e-3 * rng.normal(size=9)
    dq = np.zeros((2, 12))
    dq[1, :3] = [0.01, 0.0, -0.02]
    contact_case("floor", [floor, cube], [False, True], q0, dq, 1e-2, 1e4, 0.5, 1000.0, 1e8, 0.01, rng,
                 out)
    # icosphere cluster on a floor: 2x2x2 level-1 spheres at ~d_hat/2 gaps
    ico = rshapes.icosphere_mesh(0.5, 1)
    meshes, dyn, qs = [floor], [False], [rb.BodyCoords.identity().q]
    for k in range(2):
        for j in range(2):
            for i in range(2):
                meshes.append(ico)
                dyn.append(True)
                A = scenes.random_rotation(rng)
                qs.append(np.concatenate([[(i - 0.5) * 1.004, (j - 0.5) * 1.004, 0.503 + k * 1.004],
                                          A.ravel()]))
    q0 = np.array(qs)
    dq = np.zeros_like(q0)
    dq[1:, :3] = rng.normal(0, 2e-3, size=(8, 3))
    dq[1:, 3:] = rng.normal(0, 1e-3, size=(8, 9))
    contact_case("ico", meshes, dyn, q0, dq, 1e-2, 1e4, 0.5, 1000.0, 1e8, 0.01, rng, out)
    save("contact.npz", out)


# ---------------------------------------------------------------------------
def gen_box_stack(steps=100):
    spec = scenes.box_stack(seed=0, steps=steps)
    model = ref_model(spec.meshes, spec.dynamic, spec.density, spec.kappa_ortho)
    params = rs.StepParams(**spec.params)
    state = rs.SimState(q=spec.q0.copy(), q_dot=spec.q_dot0.copy())
    qs, qds, its, conv, mind, ipv, ncand = [spec.q0.copy()], [spec.q_dot0.copy()], [], [], [], [], []
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(steps):
            state, st = rs.advance_step(model, state, params)
            qs.append(state.q.copy())
            qds.append(state.q_dot.copy())
            its.append(st.iterations)
            conv.append(st.converged)
            mind.append(st.min_distance)
            ipv.append(st.ip_value)
            ncand.append(st.candidates)
    el = time.perf_counter() - t0
    out = dict(q=np.array(qs), q_dot=np.array(qds), iterations=np.array(its), converged=np.array(conv),
               min_distance=np.array(mind), ip_value=np.array(ipv), candidates=np.array(ncand),
               seconds=np.array(el))
    pack_bodies("scene_", model.bodies, out)
    print(f"box stack {steps} steps: {el:.2f}s, {np.sum(its)} Newton iterations")
    save("box_stack.npz", out)


def gen_ico_pile(steps=40):
    """A 2x2x2 icosphere pile with friction (mu=0.5), level-1 spheres, 40 steps."""
    spec = scenes.icosphere_pile(seed=3, nx=2, ny=2, nz=2, steps=steps, mu=0.5, subdiv=1)
    model = ref_model(spec.meshes, spec.dynamic, spec.density, spec.kappa_ortho)
    params = rs.StepParams(**spec.params)
    state = rs.SimState(q=spec.q0.copy(), q_dot=spec.q_dot0.copy())
    qs, its, mind = [spec.q0.copy()], [], []
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(steps):
            state, st = rs.advance_step(model, state, params)
            qs.append(state.q.copy())
            its.append(st.iterations)
            mind.append(st.min_distance)
    el = time.perf_counter() - t0
    out = dict(q=np.array(qs), iterations=np.array(its), min_distance=np.array(mind), seconds=np.array(el))
    pack_bodies("scene_", model.bodies, out)
    print(f"ico pile {steps} steps: {el:.2f}s, {np.sum(its)} Newton iterations")
    save("ico_pile.npz", out)


def gen_friction_outer(pre=22, steps=8):
    """The 2x2x2 icosphere pile with friction_outer_iters=2 (solver.py:523-531): the
    lagged friction is refreshed (broad phase + friction_precompute at q) after the
    first Newton solve of each step.  `pre` ordinary steps first, so contacts exist."""
    spec = scenes.icosphere_pile(seed=3, nx=2, ny=2, nz=2, mu=0.5, subdiv=1)
    model = ref_model(spec.meshes, spec.dynamic, spec.density, spec.kappa_ortho)
    params = rs.StepParams(**spec.params)
    state = rs.SimState(q=spec.q0.copy(), q_dot=spec.q_dot0.copy())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(pre):
            state, _ = rs.advance_step(model, state, params)
        out = dict(q_start=state.q.copy(), qdot_start=state.q_dot.copy(), step_start=np.array(state.step_index),
                   time_start=np.array(state.time))
        params2 = rs.StepParams(**dict(spec.params, friction_outer_iters=2))
        qs, its = [], []
        for _ in range(steps):
            state, st = rs.advance_step(model, state, params2)
            qs.append(state.q.copy())
            its.append(st.iterations)
    out.update(q=np.array(qs), iterations=np.array(its))
    print(f"friction outer: {steps} steps, iterations {its}")
    save("friction_outer.npz", out)


def gen_trajectory(name, spec, steps):
    """Reference trajectory of a small version of a BASELINE scene (q per step, iterations, min distance)."""
    model = ref_model(spec.meshes, spec.dynamic, spec.density, spec.kappa_ortho)
    params = rs.StepParams(**spec.params)
    state = rs.SimState(q=spec.q0.copy(), q_dot=spec.q_dot0.copy())
    qs, its, mind = [spec.q0.copy()], [], []
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(steps):
            state, st = rs.advance_step(model, state, params)
            qs.append(state.q.copy())
            its.append(st.iterations)
            mind.append(st.min_distance)
    el = time.perf_counter() - t0
    out = dict(q=np.array(qs), iterations=np.array(its), min_distance=np.array(mind), seconds=np.array(el))
    pack_bodies("scene_", model.bodies, out)
    print(f"{name} {steps} steps: {el:.2f}s, {np.sum(its)} Newton iterations")
    save(name + ".npz", out)


def gen_cube_drop(steps=70):
    """Config 3 in small: 2x2x2 unit cubes (1.2 m pitch, random rotations) into the open container, mu=0.2."""
    gen_trajectory("cube_drop", scenes.cube_drop(seed=0, n=2, steps=steps), steps)


def gen_chainmail(steps=40):
    """Config 5 in small: 2 chains of 3 interlocked tori (top link fixed), mu=0.3, dt=0.005, d_hat=1e-4."""
    gen_trajectory("chainmail", scenes.chainmail(seed=0, n_chains=2, links=3, chains_x=2, steps=steps), steps)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernels", "contact", "box_stack", "ico_pile", "cube_drop", "chainmail"]
    if "kernels" in which:
        gen_kernels()
    if "contact" in which:
        gen_contact()
    if "box_stack" in which:
        gen_box_stack()
    if "ico_pile" in which:
        gen_ico_pile()
    if "friction_outer" in which:
        gen_friction_outer()
    if "cube_drop" in which:
        gen_cube_drop()
    if "chainmail" in which:
        gen_chainmail()
