"""Joint-reduction fixtures from the REFERENCE (constraints.py + solver.py:479-490).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_joints.py

Scenarios follow the reference's own constraint tests (pkg/tests/test_constraints.py):
a free proxy on a falling box (:119-153), an axis-constrained torqued prism
(:156-200), two hinged bars under gravity (:203-257), and the hinged bars with an
extra axis-anchor elimination (constrain_linear + axis_anchor_rows) on a third
body resting nearby.  Each stores the per-step q, q_dot, u, iterations and energy
traces, plus the reduction's T and q_const.  Nothing at test time reads
/root/reference.
"""
from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import stiffbody as sb  # noqa: E402
from stiffbody import constraints as rc  # noqa: E402
from stiffbody.body import torque_point_forces  # noqa: E402
from stiffbody.shapes import box_mesh, prism_mesh  # noqa: E402


def model_of(meshes, kappa=1e11, density=1000.0):
    bodies, gms, mats = [], [], []
    for m in meshes:
        gm, vol = sb.mass_matrix(m, density)
        bodies.append(sb.CollisionBody.from_mesh(m))
        gms.append(gm)
        mats.append(sb.BodyMaterial(density, kappa, vol))
    return sb.SystemModel(bodies, gms, mats)


def gravity_fn(model):
    def fn(step, t, q):
        return np.asarray([sb.external_generalized_force(model.gmass[b], [0, 0, -9.8]) for b in range(len(q))])
    return fn


def run(model, state, params, steps):
    qs, qds, us, its, traces = [], [], [], [], []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(steps):
            state, st = sb.advance_step(model, state, params)
            qs.append(state.q.copy())
            qds.append(state.q_dot.copy())
            us.append(state.u.copy() if state.u is not None else np.zeros(0))
            its.append(st.iterations)
            traces.append(np.pad(np.asarray(st.energy_trace, dtype=float), (0, params.max_newton_iters
                                                                            - len(st.energy_trace))))
    return dict(q=np.array(qs), q_dot=np.array(qds), u=np.array(us), iterations=np.array(its),
                trace=np.array(traces))


def free_tet():
    mesh = box_mesh(0.4)
    model = model_of([mesh])
    model.force_fn = gravity_fn(model)
    q0 = np.tile(sb.BodyCoords.identity().q, (1, 1))
    model.reduction = rc.build_constrained_system([True], {0: rc.make_free_tet(size=0.5)}, q0)
    state = sb.SimState(q=q0.copy(), q_dot=np.zeros((1, 12)))
    state.q_dot[0, :3] = [0.1, 0.2, 0.0]
    return model, state, sb.StepParams(dt=0.01, newton_tol=1e-11), 10


def rotor():
    mesh = prism_mesh(8, radius=0.3, height=0.2, axis=2)
    model = model_of([mesh])
    gm = model.gmass[0]

    def torque_fn(step, t, q):
        A = q[0, 3:].reshape(3, 3)
        pairs = torque_point_forces([0, 0, 2.0], A, arm_scale=0.2)
        return np.asarray([sb.external_generalized_force(gm, np.zeros(3), pairs)])

    model.force_fn = torque_fn
    q0 = np.tile(sb.BodyCoords.identity().q, (1, 1))
    tet = rc.make_axis_tet([0.1, 0.05, 0.0], [0.0, 0.0, 1.0], size=0.3)
    model.reduction = rc.build_constrained_system([True], {0: tet}, q0)
    state = sb.SimState(q=q0.copy(), q_dot=np.zeros((1, 12)))
    return model, state, sb.StepParams(dt=0.01, newton_tol=1e-6), 40


def hinge(anchor=False):
    bar = box_mesh([0.4, 0.1, 0.1])
    meshes = [bar, bar] + ([box_mesh(0.2)] if anchor else [])
    model = model_of(meshes, kappa=1e10)
    model.force_fn = gravity_fn(model)
    n = len(meshes)
    q0 = np.tile(sb.BodyCoords.identity().q, (n, 1))
    q0[1, :3] = [0.42, 0.0, 0.0]
    if anchor:
        q0[2, :3] = [0.2, 0.6, 0.0]
    hinge_world = np.array([0.21, 0.0, 0.0])
    d = np.array([0.0, 1.0, 0.0])
    ta = rc.make_axis_tet(hinge_world, d, size=0.1, fix_edge=False)
    tb = rc.make_axis_tet(hinge_world - q0[1, :3], d, size=0.1, fix_edge=False)
    ta = rc.VirtualTet(ta.rest_vertices, ta.fixed_dof_mask | np.array([False] * 3 + [True] * 3 + [False] * 3 + [True] * 3))
    tb = rc.VirtualTet(tb.rest_vertices, np.zeros(12, dtype=bool), shared_vertex_links=((1, 0, 1), (3, 0, 3)))
    red = rc.build_constrained_system([True] * n, {0: ta, 1: tb}, q0)
    if anchor:  # body 2 may only rotate about a vertical axis off its centre
        C, rhs = rc.axis_anchor_rows(2, n, [0.05, 0.0, 0.0], [0.0, 0.0, 1.0], q0[2], arm=0.1)
        red = rc.constrain_linear(red, C, rhs)
    model.reduction = red
    state = sb.SimState(q=q0.copy(), q_dot=np.zeros((n, 12)))
    if anchor:  # spin about the anchored axis: p_dot = -Omega a, A_dot = Omega (A = I)
        w = 0.5
        state.q_dot[2, :3] = [0.0, -0.05 * w, 0.0]
        state.q_dot[2, 3:] = np.array([[0.0, -w, 0.0], [w, 0.0, 0.0], [0.0, 0.0, 0.0]]).reshape(9)
        state.q_dot = (red.T @ red.extract_u_rate(state.q_dot.reshape(-1))).reshape(n, 12)
    state.u = red.extract_u(state.q[model.dyn_indices].reshape(-1))
    return model, state, sb.StepParams(dt=0.01, newton_tol=1e-6), 20


def main():
    out = {}
    for name, make in (("free", free_tet), ("rotor", rotor), ("hinge", hinge),
                       ("anchor", lambda: hinge(anchor=True))):
        model, state, params, steps = make()
        out[f"{name}_q0"] = state.q.copy()
        out[f"{name}_qd0"] = state.q_dot.copy()
        out[f"{name}_T"] = model.reduction.T
        out[f"{name}_qc"] = model.reduction.q_const
        r = run(model, state, params, steps)
        for k, v in r.items():
            out[f"{name}_{k}"] = v
        print(name, "steps", steps, "iterations", r["iterations"].tolist(), flush=True)
    path = os.path.join(HERE, "joints.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    main()
